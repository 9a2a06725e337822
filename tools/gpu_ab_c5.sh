set -u
mkdir -p gpurun_out/s18
timeout 1800 python tools/ab_variants.py --prebuilt --config C5 --steps 5 --warmup 3 base: pf: apf: both: base: pf: > gpurun_out/s18/ab.log 2>&1
echo done >> gpurun_out/s18/ab.log
