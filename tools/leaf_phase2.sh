#!/bin/bash
mkdir -p gpurun_out
python tools/trace.py c4 --every 4 --reps 2 > gpurun_out/r02_trace_c4.txt 2>&1
BR_BUILD_PROF=1 python -m paper_1709_00302_b200.build > /dev/null 2>&1 && \
for c in 256x32 2016x32 4096x32 16384x16; do BR_LEAF_PROF=1 python tools/panel_bench.py $c; done > gpurun_out/lc_phases2.txt 2>&1
cat gpurun_out/lc_phases2.txt; head -5 gpurun_out/r02_trace_c4.txt
