#!/bin/bash
# Round profiling pass (run under gpurun). Each ncu run follows a plain run of
# the same command that exited 0. Outputs land in gpurun_out/.
set -x
mkdir -p gpurun_out
CMD="python tools/one_reduction.py c4"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
    --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD1="python tools/one_reduction.py c1"
$CMD1 > gpurun_out/prof_plain1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches_c1.csv $CMD1 > gpurun_out/ncu_launch1.log 2>&1
# panel leaves: the 2D-layout leaf at c1's and c4's tail heights, the 1D leaf
# for c4's tallest panels
for c in 2016x32 4096x32; do
  CMD2="python tools/panel_bench.py $c"
  $CMD2 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:leaf2 -c 1 \
      -o gpurun_out/prof_leaf2_$c $CMD2 > gpurun_out/ncu_full_leaf2_$c.log 2>&1
done
CMD3="python tools/panel_bench.py 16384x16"
$CMD3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:leaf_reg -c 1 \
    -o gpurun_out/prof_leaf1 $CMD3 > gpurun_out/ncu_full_leaf1.log 2>&1
# dominant update kernels at c4 iteration-0 shapes
CMD4="python tools/gemm_bench.py left 16384 16128 256 1"
$CMD4 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dgemm -c 2 \
    -o gpurun_out/prof_gemm $CMD4 > gpurun_out/ncu_full_gemm.log 2>&1
ls -la gpurun_out
