python tools/gemm_bench.py left 16384 16128 256 3
python tools/gemm_bench.py right 16128 16128 256 3
python tools/gemm_bench.py symm 16384 16384 256 3
python tools/gemm_bench.py syr2k 16384 16384 256 3
python tools/gemm_bench.py left 8192 8192 128 3
python tools/gemm_bench.py symm 2016 2016 32 3
python tools/gemm_bench.py syr2k 2016 2016 32 3
python tools/gemm_bench.py left 16384 16128 256 1 > /dev/null && ncu --set full --import-source on -k regex:dgemm -c 3 -o gpurun_out/gemm_left python tools/gemm_bench.py left 16384 16128 256 1 > gpurun_out/ncu_gl.log 2>&1
python tools/gemm_bench.py syr2k 16384 16384 256 1 > /dev/null && ncu --set full --import-source on -k regex:dgemm -c 1 -o gpurun_out/gemm_syr2k python tools/gemm_bench.py syr2k 16384 16384 256 1 > gpurun_out/ncu_gs.log 2>&1
