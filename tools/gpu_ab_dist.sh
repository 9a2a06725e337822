set -u
mkdir -p gpurun_out/s12
timeout 1500 python tools/ab_variants.py --prebuilt --config C5 --steps 2 --warmup 1 --extra "--virtual-shards 8" base: dkb5: dku3: dk35: dk36: > gpurun_out/s12/ab.log 2>&1
echo done >> gpurun_out/s12/ab.log
