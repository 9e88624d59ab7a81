"""GPU kernels behind the reference `bandred.kernels` interface.

Drop-in for ref kernels.py (house_gen 86-110, qr_panel 165-208, lq_panel
211-255, build_w 139-149, apply_wy_left/right 258-309, symm_lower 312-341,
syr2k_lower 344-378, sym_two_sided_update 381-401). Inputs/outputs are
NumPy arrays with the reference's shapes and in-place semantics; the
arithmetic runs in the sm_100a library (libbandred_b200.so) through the C
ABI. `workers` arguments are accepted for signature compatibility and
ignored (the GPU decides its own tiling).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib


@dataclass
class PanelFactors:
    """Compact-WY factors: Q = I + W Y^T, W = Y T (ref kernels.py:113-136)."""

    y: np.ndarray
    t: np.ndarray
    w: np.ndarray
    r_or_l: np.ndarray
    tau: np.ndarray

    @property
    def j(self):
        return self.y.shape[0]

    @property
    def b(self):
        return self.y.shape[1]


def _as2d(a, name):
    if not isinstance(a, np.ndarray) or a.ndim != 2:
        raise ValueError(f"{name} must be a 2-D array")
    return a


def house_gen(x, device=None):
    """(v, tau, beta) with the reference's sign rule (ref kernels.py:86-110)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 1 or x.size < 1:
        raise ValueError("house_gen needs a vector of length >= 1")
    h, dev = _dev.ctx(device)
    lib = _lib.load()
    X = _dev.DevMat.from_host(x, dev)
    V = _dev.DevMat(x.size, 1, dev)
    TB = _dev.DevMat(2, 1, dev)
    _dev.call("house_gen", lib.br_house_gen, h, x.size, X.ptr, V.ptr, TB.ptr)
    tb = TB.to_host()[:, 0]
    return V.to_host()[:, 0], float(tb[0]), float(tb[1])


def _panel(P, lq, device):
    if lq:
        b, j = P.shape
    else:
        j, b = P.shape
    if j < b or b < 1:
        kind = "lq_panel needs b x j with" if lq else "qr_panel needs"
        raise ValueError(f"{kind} j >= b >= 1, got {P.shape[0]} x {P.shape[1]}")
    h, dev = _dev.ctx(device)
    lib = _lib.load()
    D = _dev.DevMat.from_host(P, dev)
    Y = _dev.DevMat(j, b, dev)
    T = _dev.DevMat(b, b, dev, zero=True)
    W = _dev.DevMat(j, b, dev)
    tau = _dev.DevMat(b, 1, dev)
    fn = lib.br_lq_panel if lq else lib.br_qr_panel
    _dev.call("lq_panel" if lq else "qr_panel", fn, h, (b if lq else j), (j if lq else b), D.ptr, D.ld,
              Y.ptr, Y.ld, T.ptr, T.ld, W.ptr, W.ld, tau.ptr)
    out = D.to_host()
    y = Y.to_host()
    # reference in-place semantics: triangle factor + reflector tails
    if lq:
        tails = np.triu(y[:, :].T, 1)  # b x j, row i holds v_i[1:]
        low = np.tril(out)
        low[:, b:] = 0.0
        P[...] = low + np.where(np.triu(np.ones_like(out), 1) > 0, tails, 0.0)
        fac = np.tril(P[:b, :b]).copy(order="F")
    else:
        up = np.triu(out)
        up[b:, :] = 0.0
        P[...] = up + np.tril(y, -1)
        fac = np.triu(P[:b, :b]).copy(order="F")
    return PanelFactors(y=y, t=T.to_host(), w=W.to_host(), r_or_l=fac, tau=tau.to_host()[:, 0])


def qr_panel(P, inner_b=16, device=None):
    """In-place Householder QR of a j x b panel (ref kernels.py:165-208)."""
    _as2d(P, "P")
    if inner_b < 1:
        raise ValueError("inner_b >= 1")
    return _panel(P, False, device)


def lq_panel(P, inner_b=16, device=None):
    """In-place Householder LQ of a b x j panel (ref kernels.py:211-255)."""
    _as2d(P, "P")
    if inner_b < 1:
        raise ValueError("inner_b >= 1")
    return _panel(P, True, device)


def build_w(Y, T, device=None):
    """W = Y T (ref kernels.py:139-149)."""
    _as2d(Y, "Y"), _as2d(T, "T")
    j, b = Y.shape
    if T.shape != (b, b):
        raise ValueError("build_w: T must be b x b")
    h, dev = _dev.ctx(device)
    lib = _lib.load()
    Yd, Td = _dev.DevMat.from_host(Y, dev), _dev.DevMat.from_host(T, dev)
    Wd = _dev.DevMat(j, b, dev)
    _dev.call("build_w", lib.br_build_w, h, j, b, Yd.ptr, Yd.ld, Td.ptr, Td.ld, Wd.ptr, Wd.ld)
    return Wd.to_host()


def apply_wy_left(A, factors, workers=None, device=None):
    """A := A + Y (W^T A), in place (ref kernels.py:258-284)."""
    _as2d(A, "A")
    j, b = factors.y.shape
    if A.shape[0] != j:
        raise ValueError(f"apply_wy_left: A has {A.shape[0]} rows, factors have j={j}")
    if A.shape[1] == 0 or j == 0:
        return A
    h, dev = _dev.ctx(device)
    lib = _lib.load()
    Ad = _dev.DevMat.from_host(A, dev)
    Yd, Wd = _dev.DevMat.from_host(factors.y, dev), _dev.DevMat.from_host(factors.w, dev)
    _dev.call("apply_wy_left", lib.br_apply_wy_left, h, j, A.shape[1], Ad.ptr, Ad.ld, Yd.ptr, Yd.ld,
              Wd.ptr, Wd.ld, b)
    A[...] = Ad.to_host()
    return A


def apply_wy_right(A, factors, workers=None, device=None):
    """A := A + (A W) Y^T, in place (ref kernels.py:287-309)."""
    _as2d(A, "A")
    j, b = factors.y.shape
    if A.shape[1] != j:
        raise ValueError(f"apply_wy_right: A has {A.shape[1]} cols, factors have j={j}")
    if A.shape[0] == 0 or j == 0:
        return A
    h, dev = _dev.ctx(device)
    lib = _lib.load()
    Ad = _dev.DevMat.from_host(A, dev)
    Yd, Wd = _dev.DevMat.from_host(factors.y, dev), _dev.DevMat.from_host(factors.w, dev)
    _dev.call("apply_wy_right", lib.br_apply_wy_right, h, A.shape[0], j, Ad.ptr, Ad.ld, Yd.ptr,
              Yd.ld, Wd.ptr, Wd.ld, b)
    A[...] = Ad.to_host()
    return A


def symm_lower(A2, W, out, workers=None, device=None):
    """out := sym(A2) W reading only A2's lower triangle (ref kernels.py:312-341)."""
    _as2d(A2, "A2"), _as2d(W, "W"), _as2d(out, "out")
    j = A2.shape[0]
    if A2.shape != (j, j) or W.shape[0] != j or out.shape != (j, W.shape[1]):
        raise ValueError("symm_lower shape mismatch")
    if j == 0:
        return out
    h, dev = _dev.ctx(device)
    lib = _lib.load()
    Ad, Wd = _dev.DevMat.from_host(A2, dev), _dev.DevMat.from_host(W, dev)
    Xd = _dev.DevMat(j, W.shape[1], dev)
    _dev.call("symm_lower", lib.br_symm_lower, h, j, W.shape[1], Ad.ptr, Ad.ld, Wd.ptr, Wd.ld,
              Xd.ptr, Xd.ld)
    out[...] = Xd.to_host()
    return out


def syr2k_lower(A2, X3, Y, c0, c1, workers=None, device=None):
    """A2[:, c0:c1] += X3 Y^T + Y X3^T on the lower triangle (ref kernels.py:344-378)."""
    _as2d(A2, "A2"), _as2d(X3, "X3"), _as2d(Y, "Y")
    j = A2.shape[0]
    if A2.shape != (j, j) or X3.shape[0] != j or Y.shape != X3.shape:
        raise ValueError("syr2k_lower shape mismatch")
    if not (0 <= c0 <= c1 <= j):
        raise ValueError("syr2k_lower bad column range")
    if c0 == c1:
        return A2
    h, dev = _dev.ctx(device)
    lib = _lib.load()
    Ad = _dev.DevMat.from_host(A2, dev)
    Xd, Yd = _dev.DevMat.from_host(X3, dev), _dev.DevMat.from_host(Y, dev)
    _dev.call("syr2k_lower", lib.br_syr2k_lower, h, j, X3.shape[1], Ad.ptr, Ad.ld, Xd.ptr, Xd.ld,
              Yd.ptr, Yd.ld, c0, c1)
    A2[...] = Ad.to_host()
    return A2


def sym_two_sided_update(A2, factors, workers=None, device=None):
    """A2 := (I + W Y^T)^T A2 (I + W Y^T), lower triangle only (ref kernels.py:381-401)."""
    _as2d(A2, "A2")
    j, b = factors.y.shape
    if A2.shape != (j, j):
        raise ValueError(f"sym_two_sided_update: A2 must be {j} x {j}")
    if j == 0 or b == 0:
        return A2
    h, dev = _dev.ctx(device)
    lib = _lib.load()
    Ad = _dev.DevMat.from_host(A2, dev)
    Yd, Wd = _dev.DevMat.from_host(factors.y, dev), _dev.DevMat.from_host(factors.w, dev)
    _dev.call("sym_two_sided_update", lib.br_sym_two_sided_update, h, j, b, Ad.ptr, Ad.ld, Yd.ptr,
              Yd.ld, Wd.ptr, Wd.ld)
    A2[...] = Ad.to_host()
    return A2
