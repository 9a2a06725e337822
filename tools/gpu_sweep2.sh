set -u
O=gpurun_out/s5
mkdir -p $O
for v in sgb2 sgb4; do PEEL_LIB=variants/libpeel_$v.so timeout 300 python bench.py --config C5s --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_C5s_$v.log 2>&1; done
for g in 20 32; do PEEL_SWEEP_GROUPS=$g timeout 300 python bench.py --config C5s --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_C5s_g$g.log 2>&1; done
PEEL_SWEEP_L2MB=60 timeout 300 python bench.py --config C5s --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_C5s_l2_60.log 2>&1
timeout 120 python tools/profile_sweep.py > $O/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_group -c 1 -o $O/prof_sweep python tools/profile_sweep.py > $O/ncu_sweep.log 2>&1
echo done > $O/done
