#!/bin/bash
# ncu evidence for one round (run under gpurun, 1 GPU):
#   launch lists (time + DRAM bytes per launch) of one solve per config (graph
#   off so every kernel is attributable), --set full captures of the top
#   kernels with source correlation.
# usage: tools/ncu_round.sh <tag>
set -x
T=${1:-r01}
O=gpurun_out/ncu_$T
mkdir -p $O
NCU="ncu --clock-control none"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
$NCU --metrics $M -c 400 --csv --log-file $O/launches_c5.csv python tools/ncu_solve.py --reps 2 > $O/launches_c5.log 2>&1
$NCU --metrics $M -c 400 --csv --log-file $O/launches_c4.csv python tools/ncu_solve.py --family wilkinson --n 262144 --reps 1 > $O/launches_c4.log 2>&1
$NCU --metrics $M -c 400 --csv --log-file $O/launches_c3.csv python tools/ncu_solve.py --family toeplitz121 --n 65536 --reps 1 > $O/launches_c3.log 2>&1
$NCU --set full --import-source on -k regex:k_levels_fused -s 1 -c 1 -o $O/fused_run python tools/ncu_solve.py --reps 2 > $O/fused.log 2>&1
$NCU --set full --import-source on -k regex:k_level_fused -s 1 -c 1 -o $O/fused_l6 python tools/ncu_solve.py --reps 2 > $O/fused6.log 2>&1
$NCU --set full --import-source on -k regex:k_leaf -s 1 -c 1 -o $O/leaf python tools/ncu_solve.py --reps 2 > $O/leaf.log 2>&1
$NCU --set full --import-source on -k regex:"k_merge_nn|k_merge_prep|k_deflated_out" -s 3 -c 3 -o $O/grid python tools/ncu_solve.py --reps 1 > $O/grid.log 2>&1
$NCU --set full --import-source on -k regex:"k_secular_warp" -s 8 -c 1 -o $O/secwarp_c3 python tools/ncu_solve.py --family toeplitz121 --n 65536 --reps 1 > $O/secwarp.log 2>&1
ls -la $O
