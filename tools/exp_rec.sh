# recursive panel splitting: correctness at small sizes, panel times, c4
BR_REC_WIDTH=32 BR_REC_MIN_ROWS=0 python -m pytest tests/test_gpu_parity.py -q -x -k "panel or reduce_tri or reduce_sym or band_svd" 2>&1 | tail -3
for v in "" "BR_REC_WIDTH=128" "BR_REC_WIDTH=64" "BR_REC_WIDTH=32"; do
  echo "=== $v"; env $v python tools/panel_bench.py 16384x256 8192x256 4096x256 32512x256 2>&1 | tail -4
done
for v in "" "BR_REC_WIDTH=128 BR_REC_MIN_ROWS=8192" "BR_REC_WIDTH=64 BR_REC_MIN_ROWS=8192" "BR_REC_WIDTH=64" "BR_REC_WIDTH=32 BR_REC_MIN_ROWS=8192"; do
  echo "=== c4 $v"; env $v python tools/trace.py c4 --every 4096 --reps 3 2>&1 | head -1
done
