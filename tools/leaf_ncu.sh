#!/bin/bash
# High-rate PC sampling of the 2D leaf (run under gpurun), 1 CTA and 16 CTAs
mkdir -p gpurun_out
for c in 256x32 2016x32; do
  python tools/panel_bench.py $c > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 --warp-sampling-max-passes 50 \
      -k regex:leaf2 -c 1 -o gpurun_out/leaf_$c python tools/panel_bench.py $c > gpurun_out/leaf_ncu_$c.log 2>&1
done
ls -la gpurun_out/leaf_*
