"""Result checks with the reference's semantics (ref oracles.py:123-154).

These are exact structural checks on returned arrays (no arithmetic of the
reduction happens here), kept so reference call sites that verify results
(`band_check(res.band, w, w) == 0.0`) work unchanged.
"""
from __future__ import annotations

import numpy as np


def band_check(B, lower_bw, upper_bw):
    """Exact max |entry| outside the band; 0.0 when the off-band set is empty."""
    B = np.asarray(B)
    m, n = B.shape
    i = np.arange(m)[:, None]
    j = np.arange(n)[None, :]
    mask = (i - j > lower_bw) | (j - i > upper_bw)
    if not mask.any():
        return 0.0
    return float(np.max(np.abs(B[mask])))


def orth_residual(Q):
    """|| Q^T Q - I ||_F."""
    Q = np.asarray(Q, dtype=np.float64)
    return float(np.linalg.norm(Q.T @ Q - np.eye(Q.shape[1])))


def spectra_match(a, b, tol):
    """Compare two sorted spectra; returns (within_tol, max_deviation)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False, float("inf")
    if a.size == 0:
        return True, 0.0
    dev = float(np.max(np.abs(a - b)))
    return dev <= tol, dev
