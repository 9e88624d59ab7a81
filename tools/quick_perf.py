"""Quick device-time probe of the reductions (development tool, not the bench).

python tools/quick_perf.py c1 c2 c4 ...   [--la 0|1] [--reps 2] [--timing]
"""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1709_00302_b200 import _lib

CFG = {
    "c1": ("sevp", 2048, 32, 32),
    "c2": ("tri", 2048, 32, 32),
    "c3": ("sevp", 8192, 128, 128),
    "c4": ("tri", 16384, 256, 256),
    "c5": ("sevp", 32768, 256, 256),
    "s4k": ("sevp", 4096, 64, 64),
    "t4k": ("tri", 4096, 64, 64),
    "s8k": ("sevp", 8192, 256, 256),
    "t8k": ("tri", 8192, 256, 256),
}

ap = argparse.ArgumentParser()
ap.add_argument("cfgs", nargs="+")
ap.add_argument("--la", type=int, default=1)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--timing", action="store_true")
args = ap.parse_args()

lib = _lib.load()
h = _lib.handle(0)
dev = torch.device("cuda", 0)
names = ["panel", "symm", "syr2k", "gemm"]
for name in args.cfgs:
    kind, n, w, b = CFG[name]
    ld = (n + 31) // 32 * 32
    g = torch.Generator(device=dev).manual_seed(1)
    A0 = torch.randn((n, ld), dtype=torch.float64, device=dev, generator=g)
    if kind == "sevp":
        A0 = (A0[:, :n] + A0[:, :n].T) * 0.5
        A0 = torch.nn.functional.pad(A0, (0, ld - n)).contiguous()
    A = torch.empty_like(A0)
    for rep in range(args.reps):
        A.copy_(A0)
        torch.cuda.synchronize()
        lib.br_set_timing(h, 1 if (args.timing and rep == args.reps - 1) else 0)
        st = _lib.BrStats()
        t0 = time.perf_counter()
        if kind == "sevp":
            rc = lib.br_reduce_sym_band(h, n, w, b, args.la, A.data_ptr(), ld, None, 0, None, st)
        else:
            rc = lib.br_reduce_tri_band(h, n, n, w, b, args.la, A.data_ptr(), ld, None, st)
        t1 = time.perf_counter()
        _lib.check(rc, name)
        gf = st.nominal_flops / (st.device_ms * 1e-3) / 1e9
        print(f"{name} {kind} n={n} w={w} b={b} la={args.la}: device {st.device_ms:.2f} ms "
              f"wall {1e3*(t1-t0):.2f} ms  {gf:.0f} GFLOP/s  launches {st.launches}", flush=True)
    if args.timing:
        for c in range(4):
            ms, fl, nl = C.c_double(), C.c_double(), C.c_int64()
            lib.br_get_timing(h, c, C.byref(ms), C.byref(fl), C.byref(nl))
            if nl.value:
                print(f"   {names[c]:6s} {ms.value:9.2f} ms  {nl.value:6d} launches  "
                      f"{fl.value / (ms.value * 1e-3) / 1e12 if ms.value else 0:.2f} TFLOP/s", flush=True)
        lib.br_set_timing(h, 0)
    del A, A0
    torch.cuda.empty_cache()
