#!/bin/bash
# Generic env-variant sweep over a bench config with the trace tool (run under gpurun):
#   CFG=c4 VARIANTS="A=1 B=2,C=3" bash tools/exp_env.sh
mkdir -p gpurun_out
CFG=${CFG:-c4}
for v in ${VARIANTS}; do
  echo "=== $v"; env ${v//,/ } python tools/trace.py $CFG --every 4096 --reps 3 2>&1 | head -1
done | tee gpurun_out/exp_env_$CFG.txt
