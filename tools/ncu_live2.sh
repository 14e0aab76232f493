#!/bin/bash
O=gpurun_out/ncu_live2
mkdir -p $O
F="ncu --clock-control none --set full --import-source on"
$F -k regex:"k_live_level" -s 6 -c 1 -o $O/live_top python tools/ncu_solve.py --reps 1 > $O/top.log 2>&1
ls -la $O
