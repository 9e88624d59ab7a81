#!/bin/bash
mkdir -p gpurun_out
for v in J L D; do
  for c in c5 c3; do
    BR_GEMM_LOWER=$v timeout 900 python bench.py --config $c --no-cpu --steps 2 > gpurun_out/lc_${c}_$v.json 2>/dev/null
  done
done
for f in gpurun_out/lc_c5_*.json gpurun_out/lc_c3_*.json; do echo $f; python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['breakdown_ms'])"; done
