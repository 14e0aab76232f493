#!/bin/bash
# Round-2 ncu evidence (run under gpurun, 1 GPU): launch lists (time + DRAM bytes
# per launch, graph off, one solve per config after a warm-up solve) and
# --set full captures of the hot kernels with source correlation.
set -x
O=gpurun_out/ncu_r02b
mkdir -p $O
NCU="ncu --clock-control none"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
$NCU --metrics $M -c 600 --csv --log-file $O/launches_c5.csv python tools/ncu_solve.py --reps 2 > $O/launches_c5.log 2>&1
$NCU --metrics $M -c 400 --csv --log-file $O/launches_c4.csv python tools/ncu_solve.py --family wilkinson --n 262144 --reps 2 > $O/launches_c4.log 2>&1
$NCU --metrics $M -c 400 --csv --log-file $O/launches_c3.csv python tools/ncu_solve.py --family toeplitz121 --n 65536 --reps 2 > $O/launches_c3.log 2>&1
F="$NCU --set full --import-source on"
$F -k regex:k_levels_fused -s 1 -c 1 -o $O/fused_run python tools/ncu_solve.py --reps 2 > $O/fused.log 2>&1
$F -k regex:"^k_secular$|k_secular<" -s 13 -c 2 -o $O/secular_lane python tools/ncu_solve.py --reps 2 > $O/seclane.log 2>&1
$F -k regex:"k_zhat$|k_zhat\(|k_rows$|k_rows\(" -s 26 -c 2 -o $O/zhat_rows python tools/ncu_solve.py --reps 2 > $O/zr.log 2>&1
$F -k regex:"k_merge_nn|k_deflated_out|k_merge_prep" -s 39 -c 3 -o $O/grid_merge python tools/ncu_solve.py --reps 2 > $O/grid.log 2>&1
$F -k regex:k_leaf -s 1 -c 1 -o $O/leaf python tools/ncu_solve.py --reps 2 > $O/leaf.log 2>&1
$F -k regex:"k_secular_warp" -s 18 -c 2 -o $O/secwarp_c3 python tools/ncu_solve.py --family toeplitz121 --n 65536 --reps 2 > $O/secwarp.log 2>&1
ls -la $O
