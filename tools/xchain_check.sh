#!/bin/bash
# xchain A/B (run under gpurun): SEVP parity tests, then c1 / c3 bench with
# the fused X-product launch on and off.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -x -q -k "sym or c1 or sevp or graph or depth or reproducible or tuning or streamed or partial or dist or cyclic" > gpurun_out/xchain_tests.log 2>&1
echo "rc=$?" >> gpurun_out/xchain_tests.log
for c in c1 c3; do
  for x in 1 0; do
    BR_XCHAIN=$x timeout 600 python bench.py --config $c --no-cpu > gpurun_out/xc_${c}_$x.json 2> gpurun_out/xc_${c}_$x.err
  done
done
tail -n 3 gpurun_out/xchain_tests.log
