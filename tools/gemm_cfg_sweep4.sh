for cfg in C A D E F B L; do
  echo -n "$cfg "; BR_GEMM_RANKB=$cfg python tools/gemm_bench.py left 16384 16128 256 3 2>&1 | tail -1
done
for cfg in L D C; do echo -n "lower $cfg "; BR_GEMM_LOWER=$cfg python tools/gemm_bench.py syr2k 16384 16384 256 3 2>&1 | tail -1; done
for cfg in L D; do echo -n "lower $cfg "; BR_GEMM_LOWER=$cfg python tools/gemm_bench.py syr2k 2016 2016 32 3 2>&1 | tail -1; done
for cfg in L D; do echo -n "lower $cfg "; BR_GEMM_LOWER=$cfg python tools/gemm_bench.py syr2k 8064 8064 128 3 2>&1 | tail -1; done
