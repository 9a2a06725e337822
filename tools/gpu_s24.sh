set -u
O=gpurun_out/s25
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_multirank.py -x -q > $O/pytest.log 2>&1
echo "rc $?" >> $O/pytest.log
timeout 600 python bench.py --config C5 --virtual-shards 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_C5_virtual8.log 2>&1
timeout 600 python bench.py --config C5 --mode dist --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_C5_dist1.log 2>&1
echo done > $O/done
