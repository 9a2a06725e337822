set -u
mkdir -p gpurun_out/s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s3/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3/pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/s3/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/s3/bench_C5.log 2>&1
timeout 600 python bench.py --config C5s --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s3/bench_C5s.log 2>&1
