#!/bin/bash
# ncu --set full of the live-tier level kernel (C5 level 4: 4096 merges; and level 10)
O=gpurun_out/ncu_live
mkdir -p $O
F="ncu --clock-control none --set full --import-source on"
$F -k regex:"k_live_level" -s 0 -c 1 -o $O/live_l6 python tools/ncu_solve.py --reps 1 > $O/l4.log 2>&1
$F -k regex:"k_live_level" -s 4 -c 1 -o $O/live_l10 python tools/ncu_solve.py --reps 1 > $O/l10.log 2>&1
ls -la $O
