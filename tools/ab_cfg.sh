#!/bin/bash
# A/B of the in-tree library vs BRGPU_LIB variants on a few configs: tools/ab_cfg.sh libA.so [libB.so ...]
for cfg in "sym-uniform 1048576" "sym-uniform 4096" "wilkinson 262144" "toeplitz121 65536"; do
  python tools/ab_bench.py $cfg
  for v in "$@"; do BRGPU_LIB=$v python tools/ab_bench.py $cfg; done
done
