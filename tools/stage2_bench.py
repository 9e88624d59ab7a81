"""Second-stage timing (device events around the C-ABI call on a resident
band): band -> tridiagonal / bidiagonal at the c1 / c2 / c3 bandwidths.

    python tools/stage2_bench.py > gpurun_out/stage2_bench.txt
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1709_00302_b200 import _lib  # noqa: E402


def band(n, w, sym, seed):
    g = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(seed))
    i = torch.arange(n, device="cuda")
    keep = ((i[:, None] - i[None, :]).abs() <= w) if sym else ((i[None, :] - i[:, None] >= 0) & (i[None, :] - i[:, None] <= w))
    g = torch.where(keep, g, torch.zeros((), dtype=torch.float64, device="cuda"))
    if sym:
        g = (g + g.T) / 2
    return g.T.contiguous()  # (col, row) = column-major


def main():
    lib = _lib.load()
    h = _lib.handle(0)
    st = torch.cuda.Stream()
    lib.br_set_streams(h, C.c_void_p(st.cuda_stream), None)
    for n, w in [(2048, 32), (8192, 32), (8192, 64), (8192, 128), (16384, 64)]:
        for sym in (True, False):
            A0 = band(n, w, sym, n + w)
            d = torch.empty(n, dtype=torch.float64, device="cuda")
            e = torch.empty(n, dtype=torch.float64, device="cuda")
            times = []
            for rep in range(3):
                A = A0.clone()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                rc = (lib.br_band_to_tridiag(h, n, w, A.data_ptr(), n, d.data_ptr(), e.data_ptr()) if sym else
                      lib.br_band_to_bidiag(h, n, n, w, A.data_ptr(), n, d.data_ptr(), e.data_ptr()))
                e1.record(st)
                _lib.check(rc, "stage2")
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            flops = 6.0 * n * n * w if sym else 8.0 * n * n * w
            ms = min(times)
            print(f"{'tridiag' if sym else 'bidiag '} n={n:6d} w={w:4d}: {ms:9.2f} ms  "
                  f"({flops / ms / 1e9:.1f} GFLOP/s at ~{'6' if sym else '8'} n^2 w flops)", flush=True)


if __name__ == "__main__":
    main()
