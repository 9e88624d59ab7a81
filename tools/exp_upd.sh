#!/bin/bash
# c4 (and c3 with CFG=c3) with the overlapped update rest confined to all but N SMs
# below a trailing-rows threshold (BR_UPD_SMS / BR_UPD_ROWS); run under gpurun
mkdir -p gpurun_out
CFG=${CFG:-c4}
for v in ${VARIANTS:-"BR_UPD_SMS=0" "BR_UPD_SMS=16" "BR_UPD_SMS=32" "BR_UPD_SMS=16,BR_UPD_ROWS=8192" "BR_UPD_SMS=32,BR_UPD_ROWS=8192" "BR_UPD_SMS=32,BR_UPD_ROWS=12288" "BR_UPD_SMS=48,BR_UPD_ROWS=8192"}; do
  echo "=== $v"; env ${v//,/ } python tools/trace.py $CFG --every 4096 --reps 3 2>&1 | head -1
done | tee gpurun_out/exp_upd_$CFG.txt
