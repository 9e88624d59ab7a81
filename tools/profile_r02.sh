#!/bin/bash
# Round-2 profiling pass (run under gpurun). Each ncu run follows a plain run
# of the same command that exited 0. Outputs land in gpurun_out/.
set -x
mkdir -p gpurun_out
for c in c4 c2 c1; do
  CMD="python tools/one_reduction.py $c"
  $CMD > gpurun_out/r02_plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
      --log-file gpurun_out/r02_launches_$c.csv $CMD > gpurun_out/r02_ncu_launch_$c.log 2>&1
done
# dominant update kernel at the c4 iteration-0 shape (rank-b update)
CMD4="python tools/gemm_bench.py left 16384 16128 256 1"
$CMD4 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dgemm -c 2 \
    -o gpurun_out/r02_full_gemm_c4 $CMD4 > gpurun_out/r02_ncu_full_gemm.log 2>&1
# second stage at c1's bandwidth
python tools/stage2_bench.py > gpurun_out/stage2_bench.txt 2>&1
CMD5="python tools/stage2_bench.py"
ncu --set full --clock-control none --import-source on -k regex:sb2st -c 1 \
    -o gpurun_out/r02_full_sb2st $CMD5 > gpurun_out/r02_ncu_full_sb2st.log 2>&1
python tools/trace.py c2 --every 8 --reps 3 > gpurun_out/r02_trace_c2.txt 2>&1
ls -la gpurun_out
