#!/bin/bash
# Final round-2 evidence (1 GPU): bench lines for every config + the reference arm,
# the C5 launch list (time + DRAM bytes per launch) and --set full captures of the
# live-tier level kernel (first live level and a few-merge top level).
O=gpurun_out/final
mkdir -p $O
for c in c5 c1 c3 c4 c4s c2; do
  python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
python bench.py --impl reference > $O/bench_ref_c5.json 2> $O/bench_ref_c5.err
NCU="ncu --clock-control none"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
$NCU --metrics $M -c 600 --csv --log-file $O/launches_c5.csv python tools/ncu_solve.py --reps 2 > $O/launches_c5.log 2>&1
F="$NCU --set full --import-source on"
$F -k regex:"k_live_level" -s 0 -c 1 -o $O/live_first python tools/ncu_solve.py --reps 1 > $O/live1.log 2>&1
$F -k regex:"k_live_top" -c 1 -o $O/live_top python tools/ncu_solve.py --reps 1 > $O/live2.log 2>&1
$F -k regex:"k_live_init|k_live_bucket|k_live_scatter" -c 3 -o $O/live_aux python tools/ncu_solve.py --reps 1 > $O/live3.log 2>&1
ls -la $O
