#!/bin/bash
mkdir -p gpurun_out
for v in J D L; do
  BR_GEMM_LOWER=$v timeout 900 python bench.py --config c1 --no-cpu > gpurun_out/lc2_c1_$v.json 2>/dev/null
done
timeout 900 python bench.py --config c1 --no-cpu > gpurun_out/lc2_c1_default.json 2>/dev/null
for f in gpurun_out/lc2_c1_*.json; do echo $f; python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['breakdown_ms'])"; done
