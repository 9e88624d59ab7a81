#!/bin/bash
# High-rate PC sampling of the 2D leaf (run under gpurun), 1 CTA and 8 CTAs
mkdir -p gpurun_out
for c in 256x32 2016x32; do
  python tools/panel_bench.py $c > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on --sampling-interval 0 --sampling-max-passes 20 \
      -k regex:leaf2 -c 1 -o gpurun_out/leaf_$c python tools/panel_bench.py $c > gpurun_out/leaf_ncu_$c.log 2>&1
done
BR_BUILD_PROF=1 python -m paper_1709_00302_b200.build > /dev/null 2>&1 && \
for c in 256x32 2016x32 4096x32; do BR_LEAF_PROF=1 python tools/panel_bench.py $c; done > gpurun_out/leaf_phases.txt 2>&1
ls -la gpurun_out/leaf_*; cat gpurun_out/leaf_phases.txt
