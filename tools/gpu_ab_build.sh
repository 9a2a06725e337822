set -u
mkdir -p gpurun_out/s21
timeout 1800 python tools/ab_variants.py --prebuilt --config C5 --steps 5 --warmup 3 base: cd768: ck5b3: fe1k: > gpurun_out/s21/ab.log 2>&1
echo done >> gpurun_out/s21/ab.log
