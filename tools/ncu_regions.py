"""Per-region stall breakdown of an ncu SASS source CSV (regions split at BAR instructions)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
end = hi[1] - 1 if len(hi) > 1 else len(rows)
hdr = rows[hi[0]]
data = [r for r in rows[hi[0] + 1:end] if len(r) == len(hdr)]
iS = hdr.index("Warp Stall Sampling (All Samples)")
stalls = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: hdr.index(c) for c in stalls}
tot = sum(int(r[iS]) for r in data)
marks = [i for i, r in enumerate(data) if "BAR" in r[1] and "ERRBAR" not in r[1]]
prev = 0
for m in marks + [len(data)]:
    seg = data[prev:m + 1]
    s = sum(int(r[iS]) for r in seg)
    if s > tot * 0.01:
        br = {c: sum(int(r[idx[c]] or 0) for r in seg) for c in stalls}
        top = sorted(br.items(), key=lambda kv: -kv[1])[:5]
        print(f"[{prev:5d},{m:5d}] {100*s/tot:5.1f}%  " + "  ".join(f"{k[6:]}={100*v/max(1,s):.0f}%" for k, v in top))
    prev = m + 1
