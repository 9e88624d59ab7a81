#!/bin/bash
# Phase counters of the leaf with pair steps off / on (run under gpurun)
mkdir -p gpurun_out
export PYTHONPATH=.
BR_BUILD_PROF=1 python -m paper_1709_00302_b200.build > /dev/null 2>&1
for c in ${SHAPES:-2016x32 4096x32 8192x32 16384x16}; do
  for pm in 0 1; do echo "== $c pair=$pm"; BR_LEAF_PAIR=$pm BR_LEAF_PROF=1 python tools/panel_bench.py $c; done
done > gpurun_out/pair_phases.txt 2>&1
cat gpurun_out/pair_phases.txt
