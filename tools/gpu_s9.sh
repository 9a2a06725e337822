set -u
O=gpurun_out/s9
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_kcore.py -x -q -k "dist or narrow or host or shard" > $O/pytest.log 2>&1
echo "rc $?" >> $O/pytest.log
timeout 600 python bench.py --config C5 --virtual-shards 8 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_C5_virtual8.log 2>&1
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C5.log 2>&1
echo done > $O/done
