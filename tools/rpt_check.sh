#!/bin/bash
# Regression check of the hot kernels, then the 2D leaf with 4 rows per
# thread (BR_LEAF_RPT=4) vs 8 (run under gpurun)
mkdir -p gpurun_out
for c in c4 c5 c1; do
  timeout 900 python bench.py --config $c --no-cpu > gpurun_out/reg_${c}.json 2> gpurun_out/reg_${c}.err
done
{
for v in "" "BR_LEAF_RPT=4"; do
  echo "=== [$v]"
  env $v python tools/panel_bench.py 256x32 2016x32 4096x32 8192x32 256x16 4096x16 8064x128 4096x256 2>&1
done
} > gpurun_out/rpt_panels.txt
BR_LEAF_RPT=4 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/rpt_parity.log 2>&1; echo "rc=$?" >> gpurun_out/rpt_parity.log
for c in c1 c2 c3; do
  BR_LEAF_RPT=4 timeout 600 python bench.py --config $c --no-cpu > gpurun_out/rpt_${c}.json 2>/dev/null
done
cat gpurun_out/rpt_panels.txt; tail -2 gpurun_out/rpt_parity.log
for f in gpurun_out/reg_c*.json gpurun_out/rpt_c*.json; do echo $f; python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['breakdown_ms'])"; done
