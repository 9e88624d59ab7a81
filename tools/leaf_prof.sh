# Leaf phase counters (cycles per column step), profiling build on the box
BR_BUILD_PROF=1 python -m paper_1709_00302_b200.build > /dev/null 2>&1 || { echo build failed; exit 1; }
for c in 256x32 2016x32 4096x32 8192x32 16384x16 4096x256 16384x256; do
  BR_LEAF_PROF=1 python tools/panel_bench.py $c
done
