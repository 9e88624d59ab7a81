#!/bin/bash
# Bench every BASELINE config once (run under gpurun); JSON lines to gpurun_out/.
mkdir -p gpurun_out
for c in c4 c1 c2 c3 c5 b4; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_c4.json 2> gpurun_out/bench_ref.err
tail -n 1 gpurun_out/bench_*.json
