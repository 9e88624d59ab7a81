"""How much a concurrent panel factorization slows the rank-b update GEMM.

python tools/overlap_bench.py
Times E += Y Z (16384 x 16128, K = 256) on the main stream alone and while
the panel stream (high priority) factors panels back to back.
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
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -5)
panel = torch.cuda.Stream(device=dev, priority=-5)
lib.br_set_streams(h, C.c_void_p(main.cuda_stream), C.c_void_p(panel.cuda_stream))


def pad(n):
    return (n + 31) // 32 * 32


rows, cols, b = 16384, 16128, 256
A = torch.randn((cols, pad(rows)), dtype=torch.float64, device=dev)
Y = torch.randn((b, pad(rows)), dtype=torch.float64, device=dev)
Z = torch.randn((cols, b), dtype=torch.float64, device=dev)  # b x cols col-major, ld = b


def gemm():
    lib.br_stream_select(h, 0)
    _lib.check(lib.br_gemm(h, 0, 0, rows, cols, b, 1.0, Y.data_ptr(), pad(rows), Z.data_ptr(), b,
                           1.0, A.data_ptr(), pad(rows)), "gemm")


def panels(kind, n):
    j, pb = kind
    P0 = torch.randn((pb, pad(j)), dtype=torch.float64, device=dev)
    Yp = torch.empty_like(P0)
    Wp = torch.empty_like(P0)
    T = torch.empty((pb, pb), dtype=torch.float64, device=dev)
    tau = torch.empty(pb, dtype=torch.float64, device=dev)
    lib.br_stream_select(h, 1)
    for _ in range(n):
        _lib.check(lib.br_qr_panel(h, j, pb, P0.data_ptr(), pad(j), Yp.data_ptr(), pad(j),
                                   T.data_ptr(), pb, Wp.data_ptr(), pad(j), tau.data_ptr()), "qr")
    lib.br_stream_select(h, 0)


def small_gemms(n):
    """Zs = Y^T P_rest shapes (16 x 240, K = 16384) back to back on the panel stream."""
    Yp = torch.randn((16, pad(16384)), dtype=torch.float64, device=dev)
    Pp = torch.randn((240, pad(16384)), dtype=torch.float64, device=dev)
    Zp = torch.empty((240, 16), dtype=torch.float64, device=dev)
    lib.br_stream_select(h, 1)
    for _ in range(n):
        _lib.check(lib.br_gemm(h, 1, 0, 16, 240, 16384, 1.0, Yp.data_ptr(), pad(16384), Pp.data_ptr(),
                               pad(16384), 0.0, Zp.data_ptr(), 16), "gemm")
    lib.br_stream_select(h, 0)


e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for label, kind, n in [("alone", None, 0), ("+ 16384x16 leaves", (16384, 16), 80),
                       ("+ 2016x32 leaves", (2016, 32), 60),
                       ("+ 16384x256 panels", (16384, 256), 3), ("+ 4096x256 panels", (4096, 256), 5),
                       ("+ small split-K gemms", "gemm", 300)]:
    torch.cuda.synchronize()
    gemm()
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    p0.record(panel)
    if kind == "gemm":
        small_gemms(n)
    elif kind:
        panels(kind, n)
    p1.record(panel)
    gemm()
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    pms = p0.elapsed_time(p1) if kind else 0.0
    print(f"rank-b update {label:24s}: {ms:.3f} ms  {2 * rows * cols * b / ms / 1e9:.2f} TFLOP/s"
          f"  (panel stream busy {pms:.3f} ms)", flush=True)
