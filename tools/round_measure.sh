#!/bin/bash
# End-of-round measurements on one B200 (run under gpurun from the repo root):
# bench lines for every config, the C5 launch list (ncu, one pass) and ncu --set full captures
# of the C5 kernels.  Outputs under gpurun_out/r02/.
set -u
O=${OUT:-gpurun_out/r02}
mkdir -p $O
P="python tools/profile_step.py --n 1000000000 --c 0.75 --r 3 --k 2 --seed 6 --warm 0"
timeout 400 python bench.py > $O/bench_C5.log 2>&1
for c in C1 C2 C3 C4a C4b; do timeout 300 python bench.py --config $c > $O/bench_$c.log 2>&1; done
timeout 600 python bench.py --config C5s --steps 1 --warmup 1 > $O/bench_C5s.log 2>&1
timeout 600 python bench.py --config C5 --virtual-shards 8 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_C5_virtual8.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_C5_reference.log 2>&1
timeout 120 $P > $O/plain.log 2>&1 && \
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $O/launches_C5.csv $P > $O/ncu_launches.log 2>&1
M=lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum
timeout 600 ncu --set full --clock-control none --import-source on --metrics $M -k regex:"bin_partition|cbuild" -c 2 \
  -o $O/prof_build $P > $O/ncu_build.log 2>&1
PEEL_ROUNDS_PER_SYNC=1 timeout 600 ncu --set full --clock-control none --import-source on --metrics $M -k regex:"ckill|capply" -s 6 -c 2 \
  -o $O/prof_round4 $P > $O/ncu_round4.log 2>&1
echo done > $O/done
