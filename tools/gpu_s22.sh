set -u
O=gpurun_out/s22
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_iblt.py tests/test_gpu_iblt_forged.py tests/test_gpu_dist.py -x -q -k "iblt" > $O/pytest.log 2>&1
echo "rc $?" >> $O/pytest.log
timeout 300 python bench.py --config C2 --no-cpu-baseline > $O/bench_C2.log 2>&1
echo done > $O/done
