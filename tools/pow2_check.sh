#!/bin/bash
mkdir -p gpurun_out
{
for v in "BR_LEAF_POW2=1" ""; do
  echo "=== [$v]"
  env $v python tools/panel_bench.py 300x32 600x32 1100x32 1500x32 2016x32 3000x32 5000x32 1500x16 9000x16 2>&1
done
} > gpurun_out/pow2_panels.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pow2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pow2_parity.log
for c in c1 c2 c3 c4; do
  for v in 1 0; do
    BR_LEAF_POW2=$v timeout 900 python bench.py --config $c --no-cpu > gpurun_out/pow2_${c}_$v.json 2>/dev/null
  done
done
cat gpurun_out/pow2_panels.txt; tail -2 gpurun_out/pow2_parity.log
for f in gpurun_out/pow2_c*.json; do echo $f; python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['breakdown_ms'])"; done
