#!/bin/bash
# GPU check pass (run under gpurun): full -m gpu suite, then the default bench
# and the reference arm. Outputs land in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 2400 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for c in ${BENCH_CONFIGS:-c4}; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
if [ -n "$BENCH_REF" ]; then
  timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 1 gpurun_out/bench_*.json
