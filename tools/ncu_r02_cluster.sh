#!/bin/bash
# Round-2 evidence after the cluster live tier (1 GPU): bench lines for every
# config + the reference arm, C3/C4/C5 launch lists (time + DRAM bytes per
# launch) and a --set full capture of the cluster live-level kernel.
O=gpurun_out/r02c
mkdir -p $O
for c in c5 c1 c3 c4 c4s c2; do
  python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
python bench.py --impl reference > $O/bench_ref_c5.json 2> $O/bench_ref_c5.err
NCU="ncu --clock-control none"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
$NCU --metrics $M -c 600 --csv --log-file $O/launches_c5.csv python tools/ncu_solve.py --reps 2 > $O/launches_c5.log 2>&1
$NCU --metrics $M -c 900 --csv --log-file $O/launches_c3.csv python tools/ncu_solve.py --family toeplitz121 --n 65536 --reps 2 > $O/launches_c3.log 2>&1
$NCU --metrics $M -c 900 --csv --log-file $O/launches_c4.csv python tools/ncu_solve.py --family wilkinson --n 262144 --reps 2 > $O/launches_c4.log 2>&1
F="$NCU --set full --import-source on"
$F -k regex:"k_live_cluster" -s 2 -c 1 -o $O/k_live_cluster python tools/ncu_solve.py --reps 1 > $O/cl.log 2>&1
$F -k regex:"k_live_flow" -c 1 -o $O/k_live_flow python tools/ncu_solve.py --reps 1 > $O/fl.log 2>&1
ls -la $O
