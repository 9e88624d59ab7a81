#!/bin/bash
# Final round-2 profiling pass (run under gpurun). Each ncu run follows a plain
# run of the same command that exited 0. Outputs land in gpurun_out/.
mkdir -p gpurun_out
export PYTHONPATH=.
for c in c4 c2 c1; do
  CMD="python tools/one_reduction.py $c"
  $CMD > gpurun_out/r02f_plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
      --log-file gpurun_out/r02f_launches_$c.csv $CMD > gpurun_out/r02f_ncu_launch_$c.log 2>&1
done
# dominant update kernel at the c4 iteration-0 shape (rank-b update): traffic, DMMA pipe
CMD4="python tools/gemm_bench.py left 16384 16128 256 1"
$CMD4 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dgemm -c 2 -f \
    -o gpurun_out/r02f_full_gemm_c4 $CMD4 > gpurun_out/r02f_ncu_full_gemm.log 2>&1
# the pair-step leaf (c1 / c2's first panel) and the 1-CTA leaf with the T warp
for c in 2016x32 256x32 4096x32; do
  python tools/panel_bench.py $c > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 --warp-sampling-max-passes 50 \
      -k regex:leaf2 -c 1 -f -o gpurun_out/r02f_leaf_$c python tools/panel_bench.py $c > gpurun_out/r02f_ncu_leaf_$c.log 2>&1
done
python tools/trace.py c4 --every 4 --reps 3 > gpurun_out/r02f_trace_c4.txt 2>&1
python tools/trace.py c3 --every 4 --reps 3 > gpurun_out/r02f_trace_c3.txt 2>&1
ls -la gpurun_out | grep r02f
