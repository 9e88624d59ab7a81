#!/bin/bash
# SYMM tile configuration sweep on a SEVP config (BR_GEMM_SYMM); run under gpurun
mkdir -p gpurun_out
CFG=${CFG:-c3}
for t in ${TILES:-K J D G C E A H F B}; do
  echo "=== BR_GEMM_SYMM=$t"; BR_GEMM_SYMM=$t python tools/trace.py $CFG --every 4096 --reps 3 2>&1 | head -1
done | tee gpurun_out/exp_symm_$CFG.txt
