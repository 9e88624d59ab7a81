#!/bin/bash
# Round-2 batch (run under gpurun): stage-2 tests and timings, then the c4
# panel-mode experiments (green-context SM partition, recursive panel split).
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 600 python -m pytest tests/test_stage2.py -m gpu -q -x > gpurun_out/s2_rep$i.log 2>&1; echo "rc=$?" >> gpurun_out/s2_rep$i.log
done
python tools/stage2_bench.py > gpurun_out/stage2_bench.txt 2>&1
{
for v in "" "BR_GREEN_SMS=16" "BR_GREEN_SMS=16 BR_GREEN_ROWS=10240" "BR_GREEN_SMS=32" "BR_GREEN_SMS=32 BR_GREEN_ROWS=6144" "BR_REC_WIDTH=128 BR_REC_MIN_ROWS=8192" "BR_REC_WIDTH=64"; do
  echo "=== c4 [$v]"; env $v timeout 300 python tools/trace.py c4 --every 100000 --reps 3 2>&1 | head -1
done
} > gpurun_out/exp_c4_modes.txt 2>&1
tail -n 2 gpurun_out/s2_rep*.log; cat gpurun_out/stage2_bench.txt gpurun_out/exp_c4_modes.txt
