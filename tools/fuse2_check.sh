#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_factors.py tests/test_gpu_dist.py -m gpu -q -x > gpurun_out/f2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/f2_parity.log
for c in c1 c3; do
  for v in 1 0; do
    BR_FUSE_SMALL=$v timeout 900 python bench.py --config $c --no-cpu > gpurun_out/f2_${c}_$v.json 2>/dev/null
  done
done
bash tools/s2_threads.sh > /dev/null 2>&1
tail -2 gpurun_out/f2_parity.log; cat gpurun_out/s2_threads.txt; tail -2 gpurun_out/s2_t32.log
for f in gpurun_out/f2_c*.json; do echo $f; python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['breakdown_ms'])"; done
