set -u
O=gpurun_out/s8
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q  > $O/pytest_dist.log 2>&1
echo "rc $?" >> $O/pytest_dist.log
timeout 600 python bench.py --config C5 --virtual-shards 8 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_C5_virtual8.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:shard_filter -c 1 -o $O/prof_filter python bench.py --config C5 --virtual-shards 8 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu.log 2>&1
echo done > $O/done
