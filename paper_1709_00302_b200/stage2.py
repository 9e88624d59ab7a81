"""Second stage of the two-stage reductions: the band
the first stage returns -> symmetric tridiagonal (SEVP) or upper bidiagonal
(SVD), by Householder bulge chasing on the GPU (csrc/stage2.cu).

The reference package stops at the band (the
paper motivates the second stage), so these are extensions
with no reference counterpart. The eigenvalues (singular values) of the
result are those of the band; together with reduce_sym_band /
reduce_tri_band they complete the dense -> tridiagonal / bidiagonal
pipeline. Bandwidth w <= 128.

    res = bandred.reduce_sym_band(A, bandred.SevpConfig(n, 32, 32))
    d, e = bandred.band_to_tridiagonal(res.band, 32)
"""
from __future__ import annotations

import numpy as np

from . import _dev, _lib


def _check_w(w):
    if not 1 <= int(w) <= 128:
        raise ValueError("the second stage handles bandwidths 1 <= w <= 128")


def band_to_tridiagonal(band: np.ndarray, w: int, device=None):
    """Symmetric band (bandwidth w; the lower triangle is read) ->
    (d, e): diagonal (n) and subdiagonal (n - 1) of an orthogonally similar
    symmetric tridiagonal matrix. The input is not modified."""
    band = np.asarray(band, dtype=np.float64)
    if band.ndim != 2 or band.shape[0] != band.shape[1]:
        raise ValueError("band_to_tridiagonal needs a square matrix")
    _check_w(w)
    n = band.shape[0]
    if n == 0:
        return np.zeros(0), np.zeros(0)
    h, dev = _dev.ctx(device)
    lib = _lib.load()
    A = _dev.DevMat.from_host(band, dev)
    D = _dev.DevMat(n, 1, dev)
    E = _dev.DevMat(max(n - 1, 1), 1, dev)
    _dev.call("band_to_tridiag", lib.br_band_to_tridiag, h, n, int(w), A.ptr, A.ld, D.ptr, E.ptr)
    return D.to_host()[:, 0], E.to_host()[: n - 1, 0]


def band_to_bidiagonal(band: np.ndarray, w: int, device=None):
    """Upper triangular band (bandwidth w, m >= n) -> (d, e): diagonal and
    superdiagonal of an orthogonally equivalent upper bidiagonal matrix.
    m < n: the triangular-band output of a wide matrix is a LOWER band (ref
    svd.py:221-232); it is reduced through its transpose."""
    band = np.asarray(band, dtype=np.float64)
    if band.ndim != 2:
        raise ValueError("band_to_bidiagonal needs a 2-D array")
    _check_w(w)
    m, n = band.shape
    if m < n:  # the transpose of a lower band is an upper band: reduce A^T
        return band_to_bidiagonal(np.ascontiguousarray(band.T), w, device)
    if n == 0:
        return np.zeros(0), np.zeros(0)
    h, dev = _dev.ctx(device)
    lib = _lib.load()
    A = _dev.DevMat.from_host(band, dev)
    D = _dev.DevMat(n, 1, dev)
    E = _dev.DevMat(max(n - 1, 1), 1, dev)
    _dev.call("band_to_bidiag", lib.br_band_to_bidiag, h, m, n, int(w), A.ptr, A.ld, D.ptr, E.ptr)
    return D.to_host()[:, 0], E.to_host()[: n - 1, 0]
