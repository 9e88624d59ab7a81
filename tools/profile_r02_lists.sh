#!/bin/bash
# Launch lists of one reduction per config under ncu (run under gpurun), each after
# the same command exited 0 without ncu. Under ncu the SM partition is off
# (green-context streams cannot be profiled).
mkdir -p gpurun_out
export PYTHONPATH=.
for c in c4 c2 c1 c3; do
  CMD="python tools/one_reduction.py $c"
  $CMD > gpurun_out/r02f_plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
      --log-file gpurun_out/r02f_launches_$c.csv $CMD > gpurun_out/r02f_ncu_launch_$c.log 2>&1
  tail -1 gpurun_out/r02f_plain_$c.log; tail -1 gpurun_out/r02f_ncu_launch_$c.log
done
