for cfg in L A B C; do
  for shape in "left 16384 16128 256" "right 16128 16128 256" "symm 16384 16384 256" "left 8192 8064 128" "symm 8064 8064 128" "left 2048 2016 32" "symm 2016 2016 32"; do
    echo -n "$cfg "; BR_GEMM_BIG=$cfg python tools/gemm_bench.py $shape 3 2>&1 | tail -1
  done
done
