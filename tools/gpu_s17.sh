set -u
O=gpurun_out/s17
mkdir -p $O
P="python tools/profile_step.py --n 1000000000 --c 0.75 --r 3 --k 2 --seed 6 --warm 0"
M=lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum
PEEL_ROUNDS_PER_SYNC=1 timeout 600 ncu --set full --clock-control none --import-source on --metrics $M -k regex:"ckill|capply" -s 6 -c 2 -o $O/prof_round4 $P > $O/ncu_round4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --metrics $M -k regex:"bin_partition|cbuild" -c 2 -o $O/prof_build $P > $O/ncu_build.log 2>&1
echo done > $O/done
