"""Run exactly one reduction of a bench config through the C ABI (for ncu launch lists).

python tools/one_reduction.py c4
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_1709_00302_b200 import _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
kind, n, w, b, _ = bench.CONFIGS[cfg]
lib = _lib.load()
h = _lib.handle(0)
dev = torch.device("cuda", 0)
A_host = bench.make_input(cfg)
ld = (n + 31) // 32 * 32
A = torch.empty((n, ld), dtype=torch.float64, device=dev)
A[:, :n].copy_(torch.from_numpy(np.asfortranarray(A_host).T))
torch.cuda.synchronize()
st = _lib.BrStats()
if kind == "sevp":
    rc = lib.br_reduce_sym_band(h, n, w, b, 1, A.data_ptr(), ld, None, 0, None, st)
elif kind == "band":
    rc = lib.br_reduce_band(h, n, n, w, b, 1, 1, A.data_ptr(), ld, None, st)
else:
    rc = lib.br_reduce_tri_band(h, n, n, w, b, 1, A.data_ptr(), ld, None, st)
_lib.check(rc, "reduce")
print(f"{cfg}: {st.device_ms:.2f} ms, {st.launches} launches", flush=True)
