for cfg in C E F; do
  for shape in "left 16384 16128 256" "right 16128 16128 256" "left 8192 8064 128"; do
    echo -n "$cfg "; BR_GEMM_BIG=$cfg python tools/gemm_bench.py $shape 3 2>&1 | tail -1
  done
done
for cfg in A E F; do echo -n "$cfg "; BR_GEMM_SYMM=$cfg python tools/gemm_bench.py symm 16384 16384 256 3 2>&1 | tail -1; done
