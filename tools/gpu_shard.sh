set -u
O=gpurun_out/s7
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > $O/pytest_dist.log 2>&1
echo "rc $?" >> $O/pytest_dist.log
timeout 600 python bench.py --config C5 --virtual-shards 8 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_C5_virtual8.log 2>&1
PEEL_SHARD_FILTER=0 timeout 600 python bench.py --config C5 --virtual-shards 8 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_C5_virtual8_nofilter.log 2>&1
timeout 600 python bench.py --config C5 --virtual-shards 4 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_C5_virtual4.log 2>&1
echo done > $O/done
