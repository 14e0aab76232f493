#!/bin/bash
# ncu --set full of the high (latency-bound) C5 levels: lane-tier k_secular at level 9,
# warp-tier k_secular_warp at level 10 (one solve, warm L2 from the earlier kernels)
O=gpurun_out/ncu_hi
mkdir -p $O
F="ncu --clock-control none --set full --import-source on"
$F -k regex:"^k_secular$" -s 5 -c 1 -o $O/seclane_l9 python tools/ncu_solve.py --reps 1 > $O/l9.log 2>&1
$F -k regex:"^k_secular_warp$" -s 3 -c 1 -o $O/secwarp_l10 python tools/ncu_solve.py --reps 1 > $O/l10.log 2>&1
ls -la $O
