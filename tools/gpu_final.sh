set -u
mkdir -p gpurun_out/r02c
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02c/pytest_gpu.log 2>&1
echo "rc $?" >> gpurun_out/r02c/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c/smoke.log 2>&1
echo "rc $?" >> gpurun_out/r02c/smoke.log
OUT=gpurun_out/r02c bash tools/round_measure.sh
