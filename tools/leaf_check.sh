#!/bin/bash
# Leaf change check (run under gpurun): parity tests, panel timings, leaf
# phase counters, c1-c4 bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_factors.py tests/test_stage2.py -m gpu -q -x > gpurun_out/lc_parity.log 2>&1; echo "rc=$?" >> gpurun_out/lc_parity.log
python tools/panel_bench.py 256x32 2016x32 4096x32 8192x32 256x16 4096x16 16384x16 8064x128 4096x256 16384x256 > gpurun_out/lc_panels.txt 2>&1
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c --no-cpu > gpurun_out/lc_${c}.json 2> gpurun_out/lc_${c}.err
done
BR_BUILD_PROF=1 python -m paper_1709_00302_b200.build > /dev/null 2>&1 && \
for c in 256x32 2016x32 4096x32; do BR_LEAF_PROF=1 python tools/panel_bench.py $c; done > gpurun_out/lc_phases.txt 2>&1
tail -2 gpurun_out/lc_parity.log; cat gpurun_out/lc_panels.txt gpurun_out/lc_phases.txt
for f in gpurun_out/lc_c*.json; do echo $f; python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['breakdown_ms'])"; done
