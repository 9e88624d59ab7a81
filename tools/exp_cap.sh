# panel GEMMs on a capped grid (real SM-slot cap) for tall panels
for v in "" "BR_PANEL_CAP=16" "BR_PANEL_CAP=32" "BR_PANEL_CAP=64" "BR_PANEL_CAP=32 BR_PANEL_CAP_ROWS=10240" "BR_PANEL_CAP=32 BR_PANEL_CAP_ROWS=4096"; do
  echo "=== c4 $v"; env $v python tools/trace.py c4 --every 4096 --reps 3 2>&1 | head -1
done
BR_PANEL_CAP=32 BR_PANEL_CAP_ROWS=0 python -m pytest tests/test_gpu_parity.py -q -x -k "panel or reduce_tri or reduce_sym" 2>&1 | tail -2
