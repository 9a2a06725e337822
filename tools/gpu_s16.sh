set -u
O=gpurun_out/s16
mkdir -p $O
PEEL_CB_MEMSET=1 timeout 900 python -m pytest tests/test_gpu_kcore.py -x -q -k "compact_rounds_modes or host or binned or C5 or golden" > $O/pytest_memset.log 2>&1
echo "rc $?" >> $O/pytest_memset.log
for i in 1 2; do
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C5_base_$i.log 2>&1
PEEL_CB_MEMSET=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C5_memset_$i.log 2>&1
done
echo done > $O/done
