for cfg in "sym-uniform 4096" "sym-uniform 16384" "sym-uniform 65536" "toeplitz121 65536" "wilkinson 262144" "sym-uniform 1048576"; do
  python tools/ab_bench.py $cfg
  for v in tools/libfew0.so tools/libfew2.so; do BRGPU_LIB=$v python tools/ab_bench.py $cfg; done
done
