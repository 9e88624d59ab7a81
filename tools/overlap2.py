"""Interference cost of panel-stream work on the trailing-update GEMM.

python tools/overlap2.py
The main stream runs the c4 rank-b update E += Y Z (16384 x 16128, K = 256)
back to back for a fixed time; the panel stream (high priority) runs one
kind of panel work in a loop. Reported per kind: the item's time alone, its
time under the GEMM, and the GEMM time it costs per item (extra main-stream
ms / items) - the SM-time the item really takes from the update.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1709_00302_b200 import _lib

lib = _lib.load()
dev = torch.device("cuda", 0)
h = _lib.handle(0)
main = torch.cuda.Stream(device=dev, priority=0)
panel = torch.cuda.Stream(device=dev, priority=-5)
lib.br_set_streams(h, C.c_void_p(main.cuda_stream), C.c_void_p(panel.cuda_stream))


def pad(n):
    return (n + 31) // 32 * 32


rows, cols, b = 16384, 16128, 256
A = torch.randn((cols, pad(rows)), dtype=torch.float64, device=dev)
Y = torch.randn((b, pad(rows)), dtype=torch.float64, device=dev)
Z = torch.randn((cols, b), dtype=torch.float64, device=dev)


def gemm():
    lib.br_stream_select(h, 0)
    _lib.check(lib.br_gemm(h, 0, 0, rows, cols, b, 1.0, Y.data_ptr(), pad(rows), Z.data_ptr(), b,
                           1.0, A.data_ptr(), pad(rows)), "gemm")


def make_panel(j, pb):
    P0 = torch.randn((pb, pad(j)), dtype=torch.float64, device=dev)
    Yp = torch.empty_like(P0)
    Wp = torch.empty_like(P0)
    T = torch.empty((pb, pb), dtype=torch.float64, device=dev)
    tau = torch.empty(pb, dtype=torch.float64, device=dev)

    def f():
        _lib.check(lib.br_qr_panel(h, j, pb, P0.data_ptr(), pad(j), Yp.data_ptr(), pad(j),
                                   T.data_ptr(), pb, Wp.data_ptr(), pad(j), tau.data_ptr()), "qr")
    return f


def make_gemm(m, n, k, beta):
    Aa = torch.randn((k, pad(m)), dtype=torch.float64, device=dev)
    Bb = torch.randn((n, pad(k)), dtype=torch.float64, device=dev)
    Cc = torch.randn((n, pad(m)), dtype=torch.float64, device=dev)

    def f():
        _lib.check(lib.br_gemm(h, 0, 0, m, n, k, 1.0, Aa.data_ptr(), pad(m), Bb.data_ptr(), pad(k),
                               beta, Cc.data_ptr(), pad(m)), "gemm")
    return f


def make_gemm_t(m, n, k):  # C (m x n) = A^T B, A k x m, B k x n (split-K reductions)
    Aa = torch.randn((m, pad(k)), dtype=torch.float64, device=dev)
    Bb = torch.randn((n, pad(k)), dtype=torch.float64, device=dev)
    Cc = torch.empty((n, pad(m)), dtype=torch.float64, device=dev)

    def f():
        _lib.check(lib.br_gemm(h, 1, 0, m, n, k, 1.0, Aa.data_ptr(), pad(k), Bb.data_ptr(), pad(k),
                               0.0, Cc.data_ptr(), pad(m)), "gemm")
    return f


kinds = [
    ("leaf 16384x16 (16-CTA cluster)", make_panel(16384, 16)),
    ("leaf 8192x32 (16-CTA)", make_panel(8192, 32)),
    ("leaf 4096x32 (16-CTA)", make_panel(4096, 32)),
    ("leaf 2048x32 (8-CTA)", make_panel(2048, 32)),
    ("leaf 1024x32 (4-CTA)", make_panel(1024, 32)),
    ("leaf 512x32 (2-CTA)", make_panel(512, 32)),
    ("leaf 256x32 (1 CTA)", make_panel(256, 32)),
    ("rank-16 update 16384x240", make_gemm(16384, 240, 16, 1.0)),
    ("Z = Y^T P 16x240 K=16384", make_gemm_t(16, 240, 16384)),
    ("Gram 256x256 K=16384", make_gemm_t(256, 256, 16384)),
    ("panel 16384x256", make_panel(16384, 256)),
    ("panel 4096x256", make_panel(4096, 256)),
]


def timed(fn, n, stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


NG = 6
gemm()
g_alone = timed(gemm, NG, main) / NG
print(f"rank-b update alone: {g_alone:.3f} ms ({2 * rows * cols * b / g_alone / 1e9:.2f} TFLOP/s)")
for label, fn in kinds:
    lib.br_stream_select(h, 1)
    fn()
    one = timed(fn, 5, panel) / 5
    n_items = max(1, int(0.6 * NG * g_alone / one))  # keep the panel stream busy ~60 %
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    p0.record(panel)
    lib.br_stream_select(h, 1)
    for _ in range(n_items):
        fn()
    p1.record(panel)
    lib.br_stream_select(h, 0)
    for _ in range(NG):
        gemm()
    e1.record(main)
    torch.cuda.synchronize()
    g_ms = e0.elapsed_time(e1)
    p_ms = p0.elapsed_time(p1)
    cost = (g_ms - NG * g_alone) / n_items
    print(f"{label:32s}: alone {one * 1e3:8.1f} us, under GEMM {p_ms / n_items * 1e3:8.1f} us, "
          f"GEMM loses {cost * 1e3:8.1f} us per item ({cost / one:5.2f} x its own time); "
          f"GEMM {2 * rows * cols * b * NG / g_ms / 1e9:.2f} TF", flush=True)
