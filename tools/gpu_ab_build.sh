set -u
mkdir -p gpurun_out/s20
timeout 1800 python tools/ab_variants.py --prebuilt --config C5 --steps 5 --warmup 3 base: p4k4: p2k6: ru16: su8: > gpurun_out/s20/ab.log 2>&1
echo done >> gpurun_out/s20/ab.log
