#!/bin/bash
# High-rate PC sampling of the 2016 x 32 leaf with pair steps off / on (run under gpurun)
mkdir -p gpurun_out
export PYTHONPATH=.
for pm in 0 1; do
  BR_LEAF_PAIR=$pm python tools/panel_bench.py 2016x32 > /dev/null 2>&1 && \
  BR_LEAF_PAIR=$pm ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 --warp-sampling-max-passes 50 \
      -k regex:leaf2 -c 1 -f -o gpurun_out/leafp${pm}_2016x32 python tools/panel_bench.py 2016x32 > gpurun_out/leafp${pm}_ncu.log 2>&1
done
ls -la gpurun_out/leafp*
