#!/bin/bash
mkdir -p gpurun_out
{
for v in "" "BR_LEAF_RPT=44"; do
  echo "=== [$v]"
  env $v python tools/panel_bench.py 256x32 1024x32 2016x32 2048x32 256x16 2048x16 2>&1
done
} > gpurun_out/rpt44_panels.txt
BR_LEAF_RPT=44 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "panel or reduce or c1 or c2 or leaf" > gpurun_out/rpt44_parity.log 2>&1; echo "rc=$?" >> gpurun_out/rpt44_parity.log
for c in c1 c2; do
  for v in "" "BR_LEAF_RPT=44"; do
    env $v timeout 600 python bench.py --config $c --no-cpu > gpurun_out/rpt44_${c}_${v:+44}.json 2>/dev/null
  done
done
cat gpurun_out/rpt44_panels.txt; tail -2 gpurun_out/rpt44_parity.log
for f in gpurun_out/rpt44_c*.json; do echo $f; python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['breakdown_ms'])"; done
