"""Householder factors returned by the reductions (`return_factors=True`).

The reference keeps every panel's compact-WY factors only in private state
(ref sevp.py:106,128-134 `state.factors[k]`; ref svd.py:185,195 `fu` / `fv`)
and discards them. The GPU path can hand them back: the C ABI stores each
panel's Y, T and tau packed (br_factors, include/bandred_b200.h), the way
LAPACK's sytrd_sy2sb / gebrd keep their reflectors beside the band, and this
module wraps the packed arrays:

    res = reduce_sym_band(A, cfg, return_factors=True)
    f = res.factors.left[k]          # PanelFactors(y, t, w, r_or_l=None, tau)
    Q = res.factors.left.form_q()    # Q = Q_0 Q_1 ...  (A = Q B Q^T)

    tri = reduce_tri_band(A, w, b, return_factors=True)
    U = tri.factors.left.form_q(); V = tri.factors.right.form_q()   # A = U B V^T

`form_q` accumulates the block reflectors on the GPU through the C ABI
(build_w + apply_wy_right per panel, ref sevp.py:138-144's accumulate_q).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _dev, _lib
from .kernels import PanelFactors


@dataclass
class ChainFactors:
    """One reflector chain: panels (k, r0, rows, cols) stored packed.

    Panel k's Y (rows x cols, unit lower trapezoidal) is y[r0:r0+rows, k:k+cols],
    its T is t[:cols, k:k+cols] and its tau is tau[k:k+cols]. The chain's
    orthogonal factor is Q = Q_0 Q_1 ... with Q_k = I + W_k Y_k^T (embedded at
    rows/columns r0..), W_k = Y_k T_k.
    """

    y: np.ndarray
    t: np.ndarray
    tau: np.ndarray
    panels: list = field(default_factory=list)  # [(k, r0, rows, cols)]
    order: int = 0  # dimension of Q

    def keys(self):
        return [p[0] for p in self.panels]

    def __len__(self):
        return len(self.panels)

    def __contains__(self, k):
        return any(p[0] == k for p in self.panels)

    def __iter__(self):
        return iter(self.keys())

    def __getitem__(self, k) -> PanelFactors:
        for kk, r0, rows, cols in self.panels:
            if kk == k:
                y = self.y[r0:r0 + rows, k:k + cols]
                t = self.t[:cols, k:k + cols]
                return PanelFactors(y=y, t=t, w=y @ t, r_or_l=None, tau=self.tau[k:k + cols])
        raise KeyError(k)

    def form_q(self, device=None) -> np.ndarray:
        """Q = Q_0 Q_1 ... (order x order), accumulated on the GPU."""
        n = self.order
        h, dev = _dev.ctx(device)
        lib = _lib.load()
        t = _dev.torch()
        Q = _dev.DevMat(n, n, dev, zero=True)
        Q.t[:n, :n].copy_(t.eye(n, dtype=t.float64, device=dev))
        bmax = max((c for _, _, _, c in self.panels), default=1)
        Yd = _dev.DevMat(n, bmax, dev)
        Td = _dev.DevMat(bmax, bmax, dev)
        Wd = _dev.DevMat(n, bmax, dev)
        t.cuda.current_stream().synchronize()
        for k, r0, rows, cols in self.panels:
            Yd.t[:cols, :rows].copy_(t.from_numpy(np.ascontiguousarray(self.y[r0:r0 + rows, k:k + cols].T)))
            Td.t[:cols, :cols].copy_(t.from_numpy(np.ascontiguousarray(self.t[:cols, k:k + cols].T)))
            t.cuda.current_stream().synchronize()
            _lib.check(lib.br_build_w(h, rows, cols, Yd.ptr, Yd.ld, Td.ptr, Td.ld, Wd.ptr, Wd.ld),
                       "form_q")
            # Q[:, r0:r0+rows] += (Q[:, r0:r0+rows] W) Y^T
            _lib.check(lib.br_apply_wy_right(h, n, rows, Q.ptr + 8 * r0 * Q.ld, Q.ld, Yd.ptr, Yd.ld,
                                             Wd.ptr, Wd.ld, cols), "form_q")
            _lib.check(lib.br_sync(h), "form_q")
        return Q.to_host()


@dataclass
class BandFactors:
    """Factors of a reduction: `left` (QR chain; SEVP's Q, the SVD's U) and
    `right` (LQ chain, the SVD's V; None for SEVP)."""

    left: ChainFactors
    right: ChainFactors | None = None


def alloc_host(m, n, b, right):
    """Host arrays (zeroed, F-order) for the packed layout and the ctypes
    struct pointing at them."""
    yl = np.zeros((m, n), order="F")
    tl = np.zeros((b, n), order="F")
    taul = np.zeros(n)
    arrs = {"yl": yl, "tl": tl, "taul": taul}
    f = _lib.BrFactors()
    f.yl, f.ldyl, f.tl, f.ldtl, f.taul = yl.ctypes.data, m, tl.ctypes.data, b, taul.ctypes.data
    if right:
        yr = np.zeros((n, n), order="F")
        tr = np.zeros((b, n), order="F")
        taur = np.zeros(n)
        arrs.update(yr=yr, tr=tr, taur=taur)
        f.yr, f.ldyr, f.tr, f.ldtr, f.taur = yr.ctypes.data, n, tr.ctypes.data, b, taur.ctypes.data
    return f, arrs


def alloc_tau(n, right):
    """Only the reflector scalars (n doubles per chain): what the wrappers
    need for the reference-exact flop count when factors are not requested."""
    taul = np.zeros(n)
    arrs = {"taul": taul}
    f = _lib.BrFactors()
    f.taul = taul.ctypes.data
    if right:
        taur = np.zeros(n)
        arrs["taur"] = taur
        f.taur = taur.ctypes.data
    return f, arrs


def sevp_panels(n, w, b, max_iters=None):
    """(k, r0, rows, cols) of every SEVP panel (ref sevp.py:110-122, 128-134)."""
    out, k = [], 0
    while n - k - w >= 2:
        bp = min(b, n - k - w)
        out.append((k, k + w, n - k - w, bp))
        k += bp
    return out[:max_iters] if max_iters else out


def tri_panels(m, n, w, b):
    """QR and LQ panels of the triangular-band SVD (ref svd.py:179-202)."""
    left, right, k = [], [], 0
    while m - k >= 2 and k < n:
        bp = min(b, n - k, m - k)
        left.append((k, k, m - k, bp))
        jr = n - k - w
        if jr >= 1:
            right.append((k, k + w, jr, min(bp, jr)))
        k += bp
    return left, right


def band_panels(m, n, w, b):
    """QR and LQ panels of the equal-bandwidth band form (ref svd.py:265-306)."""
    left, right, k = [], [], 0
    while m - k - w >= 2 and k < n:
        bp = min(b, m - k - w, n - k)
        left.append((k, k + w, m - k - w, bp))
        jr = n - k - w
        if jr >= 1:
            right.append((k, k + w, jr, min(bp, jr)))
        k += bp
    return left, right
