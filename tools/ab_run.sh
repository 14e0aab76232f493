#!/bin/bash
# A/B device timing of library variants: tools/ab_run.sh main tools/libX.so ...
for lib in "$@"; do
  for cfg in "sym-uniform 1048576" "toeplitz121 65536" "wilkinson 262144"; do
    if [ "$lib" = main ]; then python tools/ab_bench.py $cfg 2>&1 | tail -1
    else BRGPU_LIB=$lib python tools/ab_bench.py $cfg 2>&1 | tail -1; fi
  done
done
