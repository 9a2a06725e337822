set -u
mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/s4/pytest_sweep.log 2>&1
echo "pytest rc $?" >> gpurun_out/s4/pytest_sweep.log
timeout 300 python bench.py --config C5s --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s4/bench_C5s.log 2>&1
for g in 8 12 24; do PEEL_SWEEP_GROUPS=$g timeout 300 python bench.py --config C5s --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s4/bench_C5s_g$g.log 2>&1; done
