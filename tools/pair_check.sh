#!/bin/bash
# Pair-step leaf check (run under gpurun): parity on the leaf shapes, then panel timings with pairs off / on
mkdir -p gpurun_out
export PYTHONPATH=.
timeout 600 python tools/pair_check.py > gpurun_out/pair_check.txt 2>&1; echo "rc=$?" >> gpurun_out/pair_check.txt
SH="300x32 1024x32 2016x32 4096x32 8192x32 2016x16 4096x16 16384x16 8064x128 2048x256 4096x256 16384x256"
BR_LEAF_PAIR=0 python tools/panel_bench.py $SH > gpurun_out/pair_off.txt 2>&1
BR_LEAF_PAIR=1 python tools/panel_bench.py $SH > gpurun_out/pair_on.txt 2>&1
cat gpurun_out/pair_check.txt; paste gpurun_out/pair_off.txt gpurun_out/pair_on.txt
