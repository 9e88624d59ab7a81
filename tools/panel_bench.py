"""Time br_qr_panel / br_lq_panel on device-resident panels (development tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1709_00302_b200 import _lib
lib = _lib.load(); h = _lib.handle(0); dev = torch.device("cuda", 0)
cases = [(2016, 32), (8064, 32), (8064, 128), (16384, 256), (32512, 256)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in c.split("x")) for c in sys.argv[1:]]
for j, b in cases:
    ld = (j + 31) // 32 * 32
    P0 = torch.randn((b, ld), dtype=torch.float64, device=dev)
    P = torch.empty_like(P0)
    Y = torch.empty((b, ld), dtype=torch.float64, device=dev)
    W = torch.empty_like(Y)
    T = torch.zeros((b, b), dtype=torch.float64, device=dev)
    tau = torch.empty(b, dtype=torch.float64, device=dev)
    ts = []
    for rep in range(4):
        P.copy_(P0); torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(lib.br_qr_panel(h, j, b, P.data_ptr(), ld, Y.data_ptr(), ld, T.data_ptr(), b,
                                   W.data_ptr(), ld, tau.data_ptr()), "qr")
        _lib.check(lib.br_sync(h), "sync")
        ts.append(time.perf_counter() - t0)
    if os.environ.get("BR_LEAF_PROF"):
        lib.br_leaf_prof_dump()
    print(f"qr_panel {j}x{b}: best {min(ts)*1e6:.1f} us  per column {min(ts)*1e6/b:.2f} us", flush=True)
