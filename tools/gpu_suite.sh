set -u
O=gpurun_out/r02e
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
echo "rc $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "rc $?" >> $O/smoke.log
timeout 400 python bench.py > $O/bench_C5.log 2>&1
echo done > $O/done
