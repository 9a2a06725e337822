set -u
O=gpurun_out/s19
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_multirank.py -x -q > $O/pytest.log 2>&1
echo "rc $?" >> $O/pytest.log
for i in 1 2; do timeout 600 python bench.py --config C5 --virtual-shards 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_C5_virtual8_$i.log 2>&1; done
echo done > $O/done
