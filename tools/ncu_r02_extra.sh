#!/bin/bash
# the kernel captures of tools/ncu_r02.sh whose skip counts missed (one solve each)
set -x
O=gpurun_out/ncu_r02d
mkdir -p $O
F="ncu --clock-control none --set full --import-source on"
$F -k regex:"^k_secular$" -s 0 -c 2 -o $O/secular_lane python tools/ncu_solve.py --reps 1 > $O/seclane.log 2>&1
$F -k regex:"^k_zhat$|^k_rows$" -s 0 -c 2 -o $O/zhat_rows python tools/ncu_solve.py --reps 1 > $O/zr.log 2>&1
$F -k regex:"^k_secular_warp$" -s 2 -c 1 -o $O/secwarp_c5 python tools/ncu_solve.py --reps 1 > $O/secwarp5.log 2>&1
$F -k regex:"^k_secular_warp$" -s 4 -c 1 -o $O/secwarp_c3 python tools/ncu_solve.py --family toeplitz121 --n 65536 --reps 1 > $O/secwarp3.log 2>&1
ls -la $O
