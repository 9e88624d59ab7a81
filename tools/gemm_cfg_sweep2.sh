for cfg in L D; do
  for shape in "syr2k 16384 16384 256" "syr2k 8064 8064 128" "syr2k 2016 2016 32"; do
    echo -n "$cfg "; BR_GEMM_LOWER=$cfg python tools/gemm_bench.py $shape 3 2>&1 | tail -1
  done
done
for cfg in C D; do
  for shape in "left 2048 2016 32" "right 2016 2016 32" "left 8192 8064 128"; do
    echo -n "$cfg "; BR_GEMM_BIG=$cfg python tools/gemm_bench.py $shape 3 2>&1 | tail -1
  done
done
