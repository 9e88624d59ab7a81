"""Summarize an ncu --metrics gpu__time_duration.sum launch list (CSV) by
kernel family: launches, total device time, share of the library's time.

python tools/launch_summary.py gpurun_out/launches_c4.csv [--md]
"""
import csv
import re
import sys
from collections import defaultdict


def family(name: str) -> str:
    m = re.search(r"dgemm_kernel<(\d+), (\d+), (\d+), (\d+), (\d+), (\d+), (\d+), (\d+), (\d+), (\d+)(?:, \d+)*>", name)
    if m:
        bm, bn, bk, wm, wn, st, minb, am, bmd, epi = m.groups()[:10]
        amn = {"0": "N", "1": "T", "2": "SYM"}[am]
        bmn = {"0": "N", "1": "T"}[bmd]
        epn = {"0": "gen", "1": "splitK", "2": "lower(SYR2K)"}[epi]
        return f"dgemm {bm}x{bn}x{bk} A{amn}B{bmn} {epn}"
    m = re.search(r"leaf_reg_kernel<(\d+), (\d+), (\d+)>", name)
    if m:
        return f"panel leaf (1D) NB={m.group(1)} R={m.group(2)} LT={m.group(3)}"
    m = re.search(r"leaf2_kernel<(\d+), (\d+)", name)
    if m:
        return f"panel leaf (2D) NB={m.group(1)} warps={m.group(2)}"
    for key in ("splitk_reduce", "t_assemble", "t_diag", "finalize_sym", "mask_band",
                "identity_kernel", "house_gen", "zero_fill", "copy_kernel"):
        if key in name:
            return key
    return "other (torch: inputs/copies/cuBLAS peak)"


def main():
    path = sys.argv[1]
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    iN, iV, iM = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) != len(hdr) or r[iM] != "gpu__time_duration.sum":
            continue
        f = family(r[iN])
        agg[f][0] += 1
        agg[f][1] += float(r[iV]) / 1e6  # ns -> ms
    lib = {k: v for k, v in agg.items() if not k.startswith("other")}
    tot = sum(v[1] for v in lib.values())
    md = "--md" in sys.argv
    if md:
        print("| kernel family | launches | device ms (serialised) | share of library time |")
        print("|---|---|---|---|")
    for k, (n, ms) in sorted(lib.items(), key=lambda kv: -kv[1][1]):
        if md:
            print(f"| {k} | {n} | {ms:.2f} | {100 * ms / tot:.1f} % |")
        else:
            print(f"{k:48s} {n:7d} {ms:10.2f} ms {100 * ms / tot:6.1f} %")
    o = agg.get("other (torch: inputs/copies/cuBLAS peak)")
    if o:
        print(("| " if md else "") + f"(not library: {o[0]} launches, {o[1]:.2f} ms)" + (" | | | |" if md else ""))


if __name__ == "__main__":
    main()
