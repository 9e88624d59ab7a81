#!/bin/bash
mkdir -p gpurun_out
for t in 128 256 512 1024; do echo "=== BR_S2_THREADS=$t"; BR_S2_THREADS=$t python tools/stage2_bench.py 2>&1 | head -8; done > gpurun_out/s2_threads.txt
BR_S2_THREADS=256 timeout 600 python -m pytest tests/test_stage2.py -m gpu -q -x > gpurun_out/s2_t32.log 2>&1; echo "rc=$?" >> gpurun_out/s2_t32.log
cat gpurun_out/s2_threads.txt; tail -2 gpurun_out/s2_t32.log
