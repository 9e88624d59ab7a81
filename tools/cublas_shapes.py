"""Calibrate: cuBLAS (torch) vs our DMMA GEMM on the reduction's GEMM shapes.

python tools/cublas_shapes.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1709_00302_b200 import _lib

lib = _lib.load()
h = _lib.handle(0)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(stream)
lib.br_set_streams(h, C.c_void_p(stream.cuda_stream), None)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def tm(fn, reps=4):
    fn()
    best = 1e30
    for _ in range(reps):
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


# (name, M, N, K, beta)  column-major C(MxN) = op(A) op(B) (+ beta C)
shapes = [
    ("rank-b update E += Y Z", 16384, 16128, 256, 1.0, "N", "N"),
    ("rank-b update D += Zr Yv^T", 16128, 16128, 256, 1.0, "N", "T"),
    ("reduction Z = W^T E", 256, 16128, 16384, 0.0, "T", "N"),
    ("reduction Zr = D Wv", 16128, 256, 16128, 0.0, "N", "N"),
    ("rank-b mid E += Y Z (8192)", 8192, 8064, 256, 1.0, "N", "N"),
    ("rank-b 4096", 4096, 3840, 256, 1.0, "N", "N"),
    ("rank-2b update 16384 K=512", 16384, 16128, 512, 1.0, "N", "N"),
    ("square 8192", 8192, 8192, 8192, 0.0, "N", "N"),
]
for name, M, N, K, beta, ta, tb in shapes:
    # column-major X (r x c) == torch (c x r) row-major
    A = torch.randn((K, M) if ta == "N" else (M, K), dtype=torch.float64, device=dev)
    B = torch.randn((N, K) if tb == "N" else (K, N), dtype=torch.float64, device=dev)
    Cm = torch.randn((N, M), dtype=torch.float64, device=dev)
    # cuBLAS: C^T (N x M row-major = col-major M x N) = op(B)^T op(A)^T
    Bt = B if tb == "N" else B.t()  # torch (N, K)
    At = A if ta == "N" else A.t()  # torch (K, M)
    if beta:
        f_cublas = lambda: Cm.addmm_(Bt, At)
    else:
        out = torch.empty_like(Cm)
        f_cublas = lambda: torch.mm(Bt, At, out=out)
    ms_c = tm(f_cublas)
    lda = M if ta == "N" else K
    ldb = K if tb == "N" else N
    f_ours = lambda: _lib.check(lib.br_gemm(h, int(ta == "T"), int(tb == "T"), M, N, K, 1.0, A.data_ptr(), lda,
                                            B.data_ptr(), ldb, beta, Cm.data_ptr(), M), "gemm")
    ms_o = tm(f_ours)
    fl = 2.0 * M * N * K
    print(f"{name:34s} M={M:6d} N={N:6d} K={K:6d}  cuBLAS {fl / ms_c / 1e9:7.2f} TF  ours {fl / ms_o / 1e9:7.2f} TF", flush=True)
