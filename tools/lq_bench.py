"""Time br_lq_panel (b x j row panel, transposed view inside) against br_qr_panel.

python tools/lq_bench.py [jxb ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1709_00302_b200 import _lib

lib = _lib.load()
h = _lib.handle(0)
dev = torch.device("cuda", 0)
cases = [(16384, 256), (4096, 256), (2048, 32), (8064, 128)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in c.split("x")) for c in sys.argv[1:]]
for j, b in cases:
    ldb = (b + 31) // 32 * 32
    ldj = (j + 31) // 32 * 32
    P0 = torch.randn((j, ldb), dtype=torch.float64, device=dev)  # b x j column-major, ld = ldb
    P = torch.empty_like(P0)
    Y = torch.empty((b, ldj), dtype=torch.float64, device=dev)
    W = torch.empty_like(Y)
    T = torch.zeros((b, b), dtype=torch.float64, device=dev)
    tau = torch.empty(b, dtype=torch.float64, device=dev)
    ts = []
    for rep in range(4):
        P.copy_(P0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(lib.br_lq_panel(h, b, j, P.data_ptr(), ldb, Y.data_ptr(), ldj, T.data_ptr(), b,
                                   W.data_ptr(), ldj, tau.data_ptr()), "lq")
        _lib.check(lib.br_sync(h), "sync")
        ts.append(time.perf_counter() - t0)
    print(f"lq_panel {b}x{j}: best {min(ts) * 1e6:.1f} us", flush=True)
