#!/bin/bash
# Short bench lines (run under gpurun): BENCH_CONFIGS (default c1 c2), no CPU leg
mkdir -p gpurun_out
for c in ${BENCH_CONFIGS:-c1 c2}; do
  timeout 900 python bench.py --config $c --no-cpu > gpurun_out/qb_$c.json 2> gpurun_out/qb_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/qb_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step'],3), d['breakdown_ms'])"
done
