# c4 with tall panels confined to an SM partition (green context)
for v in "" "BR_GREEN_SMS=16" "BR_GREEN_SMS=16 BR_GREEN_ROWS=10240" "BR_GREEN_SMS=16 BR_GREEN_ROWS=6144" "BR_GREEN_SMS=24" "BR_GREEN_SMS=32" "BR_GREEN_SMS=32 BR_GREEN_ROWS=6144"; do
  echo "=== $v"; env $v python tools/trace.py c4 --every 4096 --reps 3 2>&1 | head -2
done
