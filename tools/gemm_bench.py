"""Time the DMMA GEMM classes on device-resident operands (development tool).

python tools/gemm_bench.py [left|right|symm|syr2k] rows cols b [reps]
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
stream = torch.cuda.Stream(device=dev)  # a real (non-NULL) stream the library can adopt
torch.cuda.set_stream(stream)
lib.br_set_streams(h, C.c_void_p(stream.cuda_stream), None)

kind = sys.argv[1] if len(sys.argv) > 1 else "left"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
cols = int(sys.argv[3]) if len(sys.argv) > 3 else 16128
b = int(sys.argv[4]) if len(sys.argv) > 4 else 256
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5


def pad(n):
    return (n + 31) // 32 * 32


def mat(r, c):
    return torch.randn((c, pad(r)), dtype=torch.float64, device=dev)


e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if kind in ("left", "right"):
    A = mat(rows, cols)
    j = rows if kind == "left" else cols
    Y, W = mat(j, b), mat(j, b)
    fn = lib.br_apply_wy_left if kind == "left" else lib.br_apply_wy_right
    args = (h, rows, cols, A.data_ptr(), pad(rows), Y.data_ptr(), pad(j), W.data_ptr(), pad(j), b)
    flops = 4.0 * rows * cols * b
elif kind == "symm":
    A = mat(rows, rows)
    W, X = mat(rows, b), mat(rows, b)
    fn = lib.br_symm_lower
    args = (h, rows, b, A.data_ptr(), pad(rows), W.data_ptr(), pad(rows), X.data_ptr(), pad(rows))
    flops = 2.0 * rows * rows * b
else:
    A = mat(rows, rows)
    X, Y = mat(rows, b), mat(rows, b)
    fn = lib.br_syr2k_lower
    args = (h, rows, b, A.data_ptr(), pad(rows), X.data_ptr(), pad(rows), Y.data_ptr(), pad(rows), 0, rows)
    flops = 2.0 * rows * rows * b  # lower triangle of a rank-2b update
for r in range(reps):
    e0.record(stream)
    _lib.check(fn(*args), kind)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{kind} {rows}x{cols} b={b}: {ms:.3f} ms  {flops / ms / 1e9:.2f} TFLOP/s", flush=True)
