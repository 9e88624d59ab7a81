"""Summarize an ncu --page source --print-source sass CSV: hottest SASS lines."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
end = hi[1] - 1 if len(hi) > 1 else len(rows)
hdr = rows[hi[0]]
data = [r for r in rows[hi[0] + 1:end] if len(r) == len(hdr)]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
tot = sum(int(r[iS]) for r in data); totE = sum(int(r[iE]) for r in data)
print("instrs", len(data), "samples", tot, "warp-instr executed", totE)
top = sorted(range(len(data)), key=lambda i: -int(data[i][iS]))[:n]
for i in sorted(top):
    r = data[i]
    print(f"{i:5d} {int(r[iS]):7d} {int(r[iE]):9d}  {r[1].strip()}")
