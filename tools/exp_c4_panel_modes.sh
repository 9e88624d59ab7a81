for v in "" "BR_PANEL_PRIO=lo" "BR_LEAF2_WIDE=1" "BR_PERSIST_ROWS=16384" "BR_LEAF2=0"; do
  echo "=== $v"; env $v python tools/trace.py c4 --every 2048 --reps 3 2>&1 | head -3
done
