"""Flop accounting, mirroring the reference's per-call counter analytically.

The reference increments a global counter inside every `matmul` (2*m*k*n,
skipped when a dimension is 0 or alpha == 0; ref kernels.py:53-60) and
every `house_gen` (3*L; ref kernels.py:98), keyed "matmul" / "house"
(ref flops.py:12-49). The GPU path has no such per-call hook, so this module
walks the same task decomposition on the host and sums the same formulas.
A tau == 0 column (an exactly-zero panel column) makes the reference skip
a few small products; `tau_zero_correction` subtracts them given the
reductions' tau values (the wrappers fetch tau through the C ABI's factor
output), so the totals equal the reference's on every input.
"""
from __future__ import annotations

import threading

import numpy as np

SYM_STRIP = 64  # ref kernels.py:30 (syr2k strip width)


class FlopCounter:
    """Same interface as the reference's FlopCounter (ref flops.py:12-37)."""

    def __init__(self):
        self._lock = threading.Lock()
        self._by_class: dict[str, int] = {}

    def add(self, kind, amount):
        if amount <= 0:
            return
        with self._lock:
            self._by_class[kind] = self._by_class.get(kind, 0) + int(amount)

    def snapshot(self):
        with self._lock:
            out = dict(self._by_class)
        out["total"] = sum(out.values())
        return out

    @property
    def total(self):
        with self._lock:
            return sum(self._by_class.values())

    def reset(self):
        with self._lock:
            self._by_class.clear()


FLOPS = FlopCounter()


def snapshot_flops():
    return FLOPS.snapshot()


def reset_flops():
    FLOPS.reset()


class _Acc:
    def __init__(self):
        self.matmul = 0
        self.house = 0

    def mm(self, m, k, n):
        if m > 0 and k > 0 and n > 0:
            self.matmul += 2 * m * k * n

    def as_dict(self):
        d = {}
        if self.matmul:
            d["matmul"] = self.matmul
        if self.house:
            d["house"] = self.house
        d["total"] = self.matmul + self.house
        return d


def _panel(acc, j, b, inner_b=16):
    """qr_panel / lq_panel of a j x b (or b x j) panel (ref kernels.py:165-255)."""
    for s in range(0, b, inner_b):
        e = min(s + inner_b, b)
        if s > 0:
            acc.mm(s, j, e - s)
            acc.mm(s, s, e - s)
            acc.mm(j, s, e - s)
        for i in range(s, e):
            acc.house += 3 * (j - i)
            if i + 1 < e:
                acc.mm(1, j - i, e - i - 1)
                acc.mm(j - i, 1, e - i - 1)
            if i > 0:
                acc.mm(i, j - i, 1)
                acc.mm(i, i, 1)
    for i in range(b):  # build_w
        acc.mm(j, i + 1, 1)


def _syr2k(acc, j, b, c0, c1):
    """syr2k_lower strips (ref kernels.py:344-378)."""
    for s0 in range(c0, c1, SYM_STRIP):
        s1 = min(s0 + SYM_STRIP, c1)
        if s1 < j:
            acc.mm(j - s1, b, s1 - s0)
            acc.mm(j - s1, b, s1 - s0)
        for cc in range(s0, s1):
            acc.mm(s1 - cc, b, 1)
            acc.mm(s1 - cc, b, 1)


def _apply_left(acc, rows, cols, b):
    acc.mm(b, rows, cols)
    acc.mm(rows, b, cols)


def _apply_right(acc, rows, cols, b):
    acc.mm(rows, cols, b)
    acc.mm(rows, b, cols)


def sevp_counted_flops(n, w, b, variant="reference", accumulate_q=False, inner_b=16,
                       max_iters=None):
    """Reference-equivalent counted flops of reduce_sym_band (ref sevp.py:194-273);
    max_iters restricts the count to the first iterations."""
    acc = _Acc()
    ks = []
    k = 0
    while n - k - w >= 2:
        ks.append(k)
        k += min(b, n - k - w)
    for idx, k in enumerate(ks):
        if max_iters is not None and idx >= max_iters:
            break
        bp = min(b, n - k - w)
        j = n - k - w
        kn = ks[idx + 1] if idx + 1 < len(ks) else None
        bpn = min(b, n - kn - w) if kn is not None else 0
        _panel(acc, j, bp, inner_b)
        if accumulate_q:
            _apply_right(acc, n, j, bp)
        # mid block, split as the schedule splits it (apply_wy_left is
        # column-tiled, so the count is split-invariant)
        if bp < w:
            _apply_left(acc, j, w - bp, bp)
        acc.mm(j, j, bp)  # symm
        acc.mm(bp, j, bp)  # X2
        acc.mm(j, bp, bp)  # X3
        if variant == "v2" and kn is not None:
            split = max(0, bp + bpn - w)
            if split > 0:
                _syr2k(acc, j, bp, 0, split)
            if split < j:
                _syr2k(acc, j, bp, split, j)
        else:
            _syr2k(acc, j, bp, 0, j)
    return acc.as_dict(), len(ks)


def tri_counted_flops(m, n, w, b, inner_b=16, max_iters=None):
    """Reference-equivalent counted flops of reduce_tri_band (ref svd.py:179-202);
    max_iters restricts the count to the first iterations."""
    if m < n:
        m, n = n, m
    acc = _Acc()
    k = 0
    it = 0
    while m - k >= 2 and k < n:
        if max_iters is not None and it >= max_iters:
            break
        bp = min(b, n - k, m - k)
        _panel(acc, m - k, bp, inner_b)
        _apply_left(acc, m - k, n - k - bp, bp)
        jr = n - k - w
        if jr >= 1:
            bq = min(bp, jr)
            _panel(acc, jr, bq, inner_b)
            _apply_right(acc, m - k - bq, jr, bq)
        k += bp
        it += 1
    return acc.as_dict(), it


def band_counted_flops(m, n, w, b, simultaneous=False, inner_b=16):
    """Reference-equivalent counted flops of reduce_band_svd's band form
    (ref svd.py:359-391; V1 counts as Reference and V2 as Simultaneous since
    their splits are linear in the matmul dimensions)."""
    if m < n:
        m, n = n, m
    acc = _Acc()
    k = 0
    it = 0
    while m - k - w >= 2 and k < n:
        bp = min(b, m - k - w, n - k)
        jr = n - k - w
        bq = min(bp, jr) if jr >= 1 else 0
        i = m - k - w
        _panel(acc, i, bp, inner_b)
        b1end = min(k + w, n)
        if k + bp < b1end:
            _apply_left(acc, i, b1end - k - bp, bp)
        if jr >= 1:
            if not simultaneous:
                _apply_left(acc, i, jr, bp)
            _panel(acc, jr, bq, inner_b)
            if k + bq < k + w:
                _apply_right(acc, w - bq, jr, bq)
            if not simultaneous:
                _apply_right(acc, i, jr, bq)
            else:
                acc.mm(jr, i, bp)  # Z_L = D^T W_U
                acc.mm(i, jr, bq)  # Z_R = D W_V
                acc.mm(bp, jr, bq)  # Z_L^T W_V
                acc.mm(i, bp, bq)  # Y_U (.)
                acc.mm(i, bq, jr)  # X Y_V^T
                acc.mm(i, bp, jr)  # Y_U Z_L^T
        k += bp
        it += 1
    return acc.as_dict(), it


def tau_zero_correction(panels, tau, inner_b=16):
    """matmul flops the reference does NOT count for tau == 0 reflectors:
    the rank-1 update of the inner block (`if ... ti != 0.0`, ref
    kernels.py:196-201 / 244-249) and _t_extend's second product, whose
    alpha = -tau = 0 returns before counting (ref kernels.py:161, 57-60).
    panels: (k, r0, rows, cols) per panel of one chain, tau[k:k+cols] its
    reflector scalars."""
    corr = 0
    tau = np.asarray(tau)
    for k, _r0, j, bp in panels:
        for i in np.nonzero(tau[k:k + bp] == 0.0)[0]:
            i = int(i)
            e = min((i // inner_b) * inner_b + inner_b, bp)
            if i + 1 < e:
                corr += 4 * (j - i) * (e - i - 1)
            if i > 0:
                corr += 2 * i * i
    return corr


def apply_correction(flops, corr):
    """Subtract tau == 0 skips from a counted-flop dict (in place)."""
    if corr:
        flops["matmul"] = flops.get("matmul", 0) - corr
        flops["total"] = flops.get("total", 0) - corr
    return flops


def sevp_nominal_flops(n):
    """Nominal cost 4n^3/3 (ref sevp.py:92-96)."""
    if n < 0:
        raise ValueError("n >= 0")
    return round(4 * n**3 / 3)


def svd_nominal_flops(m, n):
    """Nominal cost 4(mn^2 - n^3/3), m >= n (ref svd.py:127-132)."""
    if n < 0 or m < n:
        raise ValueError("need m >= n >= 0")
    return round(4 * (m * n * n - n**3 / 3))
