"""Per-task device trace of one reduction (development tool).

python tools/trace.py c4 [--la 1] [--out gpurun_out/trace_c4.tsv] [--reps 2]

Runs the reduction with br_set_timing(h, 2) (CUDA events around every task
on its stream), writes the trace as TSV (task, stream, t0_us, t1_us) and
prints per-iteration main/panel busy time, the main stream's idle time and
the per-class totals. Tuning env vars (BR_*) apply as usual.
"""
import argparse
import collections
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1709_00302_b200 import _lib  # noqa: E402

CFG = {
    "c1": ("sevp", 2048, 32, 32), "c2": ("tri", 2048, 32, 32), "c3": ("sevp", 8192, 128, 128),
    "c4": ("tri", 16384, 256, 256), "c5": ("sevp", 32768, 256, 256), "b4": ("band", 16384, 256, 256),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--la", type=int, default=1)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--out", default=None)
    ap.add_argument("--every", type=int, default=8, help="print every k-th iteration")
    args = ap.parse_args()
    kind, n, w, b = CFG[args.cfg]
    lib = _lib.load()
    h = _lib.handle(0)
    ld = (n + 31) // 32 * 32
    g = torch.Generator(device="cuda").manual_seed(1)
    A0 = torch.rand((n, ld), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    if kind == "sevp":
        A0[:, :n] = (A0[:, :n] + A0[:, :n].T) * 0.5
    A = torch.empty_like(A0)
    st = _lib.BrStats()
    ms = []
    for rep in range(args.reps):
        A.copy_(A0)
        torch.cuda.synchronize()
        last = rep == args.reps - 1
        lib.br_set_timing(h, 2 if last else 0)
        if kind == "sevp":
            rc = lib.br_reduce_sym_band(h, n, w, b, args.la, A.data_ptr(), ld, None, 0, None, st)
        elif kind == "band":
            rc = lib.br_reduce_band(h, n, n, w, b, 1, args.la, A.data_ptr(), ld, None, st)
        else:
            rc = lib.br_reduce_tri_band(h, n, n, w, b, args.la, A.data_ptr(), ld, None, st)
        _lib.check(rc, args.cfg)
        ms.append(st.device_ms)
    rows = []
    buf = C.create_string_buffer(64)
    s, t0, t1 = C.c_int(), C.c_double(), C.c_double()
    for i in range(lib.br_trace_count(h)):
        lib.br_trace_get(h, i, buf, 64, C.byref(s), C.byref(t0), C.byref(t1))
        rows.append((buf.value.decode(), "seq" if s.value == 1 else "par", t0.value, t1.value))
    cls = {}
    names = ["panel", "symm", "syr2k", "gemm"]
    for c in range(4):
        tms, tfl, tnl = C.c_double(), C.c_double(), C.c_int64()
        lib.br_get_timing(h, c, C.byref(tms), C.byref(tfl), C.byref(tnl))
        cls[names[c]] = (tms.value, tfl.value / max(tms.value, 1e-9) / 1e9)
    lib.br_set_timing(h, 0)
    if args.out:
        with open(args.out, "w") as f:
            for r in rows:
                f.write("\t".join(str(x) for x in r) + "\n")
    it = collections.defaultdict(lambda: {"par": 0.0, "seq": 0.0, "t0": 1e18, "t1": 0.0})
    for a, sname, a0, a1 in rows:
        k = int(a.split("@")[1]) if "@" in a else -1
        it[k][sname] += (a1 - a0) / 1e3
        it[k]["t0"] = min(it[k]["t0"], a0)
        it[k]["t1"] = max(it[k]["t1"], a1)
    main = sorted((a0, a1) for _, sname, a0, a1 in rows if sname == "par")
    idle, last = 0.0, main[0][1] if main else 0.0
    for a0, a1 in main[1:]:
        if a0 > last:
            idle += a0 - last
        last = max(last, a1)
    print(f"{args.cfg} la={args.la}: device ms per rep {[round(x, 2) for x in ms]} "
          f"(traced rep {ms[-1]:.2f}); main idle {idle / 1e3:.2f} ms; "
          f"classes ms/TF: " + ", ".join(f"{k} {v[0]:.1f}/{v[1] / 1e3:.2f}" for k, v in cls.items()))
    ks = sorted(k for k in it if k >= 0)
    print("k main_ms panel_ms span_ms")
    for j, k in enumerate(ks):
        if j % args.every == 0 or j >= len(ks) - 4:
            d = it[k]
            print(k, round(d["par"], 3), round(d["seq"], 3), round((d["t1"] - d["t0"]) / 1e3, 3))


if __name__ == "__main__":
    main()
