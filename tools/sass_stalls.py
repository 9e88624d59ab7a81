"""Summarise an ncu SASS source page (--page source --csv): samples per
instruction, top stall reasons, and samples aggregated over address ranges.
Usage: ncu -i X.ncu-rep --page source --csv > s.csv; python tools/sass_stalls.py s.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
data = rows[2:]
ia, isrc, ismp = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
iex = h.index("Instructions Executed")
stall_cols = [i for i, k in enumerate(h) if k.startswith("stall_")]
tot = sum(float(r[ismp] or 0) for r in data)
print(f"total samples {tot:.0f}, instructions {len(data)}")
agg = {}
for r in data:
    for i in stall_cols:
        agg[h[i]] = agg.get(h[i], 0) + float(r[i] or 0)
print("stalls:", ", ".join(f"{k[6:]}={v:.0f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
ranked = sorted(data, key=lambda r: -float(r[ismp] or 0))[:top]
for r in ranked:
    st = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
    print(f"{r[ia]:>6} {float(r[ismp] or 0):6.0f} ex={r[iex]:>6} {r[isrc][:60]:60s} " +
          " ".join(f"{n}={v:.0f}" for v, n in st if v))
