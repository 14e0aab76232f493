set -x
O=gpurun_out/ncu_r01b
mkdir -p $O
NCU="ncu --clock-control none"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
$NCU --metrics $M -c 400 --csv --log-file $O/launches_c4.csv python tools/ncu_solve.py --family wilkinson --n 262144 --reps 1 > $O/launches_c4.log 2>&1
$NCU --metrics $M -c 400 --csv --log-file $O/launches_c3.csv python tools/ncu_solve.py --family toeplitz121 --n 65536 --reps 1 > $O/launches_c3.log 2>&1
$NCU --set full --import-source on -k regex:"k_secular_warp" -s 5 -c 1 -o $O/secwarp_c3 python tools/ncu_solve.py --family toeplitz121 --n 65536 --reps 1 > $O/secwarp.log 2>&1
$NCU --set full --import-source on -k regex:"k_rows_warp|k_zhat_warp" -s 8 -c 2 -o $O/rowszhat_c3 python tools/ncu_solve.py --family toeplitz121 --n 65536 --reps 1 > $O/rowszhat.log 2>&1
for c in c3 c4 c5; do python bench.py --config $c --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/bench_$c.json; done
ls -la $O
