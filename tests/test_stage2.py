"""Second stage (band -> tridiagonal / bidiagonal).

No reference output exists (the reference stops at the band), so the
oracle (oracle/stage2_oracle.py, the sequential task order) is pinned by
LAPACK: the eigenvalues / singular values of its result equal those of the
input, and everything off the tridiagonal / bidiagonal is exactly zero. The
GPU kernels are checked against the oracle (same reflectors: d, e agree to
rounding), against LAPACK's spectra, and against themselves run one sweep
at a time (BR_S2_CTAS=1: the sequential order) bitwise."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.stage2_oracle import sb2st, tb2bd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sym_band(n, w, seed):
    g = np.random.default_rng(seed).standard_normal((n, n))
    S = (g + g.T) / 2
    i, j = np.indices((n, n))
    S[np.abs(i - j) > w] = 0.0
    return np.asfortranarray(S)


def upper_band(m, n, w, seed):
    """Random upper band with a dominant diagonal: random triangular matrices
    are exponentially ill-conditioned, which would make d, e themselves
    ill-conditioned (the singular values stay well-conditioned either way)."""
    B = np.random.default_rng(seed).standard_normal((m, n))
    i, j = np.indices((m, n))
    B[(j < i) | (j > i + w)] = 0.0
    k = min(m, n)
    B[np.arange(k), np.arange(k)] += 3.0 * np.sqrt(w + 1.0)
    return np.asfortranarray(B)


def tri_eigs(d, e):
    return np.linalg.eigvalsh(np.diag(d) + np.diag(e, 1) + np.diag(e, -1))


def bi_svals(d, e):
    return np.linalg.svd(np.diag(d) + np.diag(e, 1), compute_uv=False)


# ---- oracle pinned by LAPACK (CPU) ------------------------------------------

@pytest.mark.parametrize("n,w", [(40, 3), (130, 32), (200, 17), (64, 63), (9, 1), (5, 4), (2, 1)])
def test_oracle_tridiagonal_preserves_spectrum(n, w):
    S = sym_band(n, w, n + w)
    d, e, W = sb2st(S, w)
    i, j = np.indices((n, n))
    assert np.all(W[np.abs(i - j) > 1] == 0.0)
    ev = np.linalg.eigvalsh(S)
    assert np.max(np.abs(tri_eigs(d, e) - ev)) <= 1e-13 * np.max(np.abs(ev))


@pytest.mark.parametrize("m,n,w", [(40, 40, 3), (140, 130, 32), (200, 200, 17), (64, 64, 63), (9, 9, 1)])
def test_oracle_bidiagonal_preserves_singular_values(m, n, w):
    B = upper_band(m, n, w, m + n + w)
    d, e, W = tb2bd(B, w)
    i, j = np.indices((n, n))
    assert np.all(W[(j != i) & (j != i + 1)] == 0.0)
    sv = np.linalg.svd(B, compute_uv=False)
    assert np.max(np.abs(bi_svals(d, e) - sv)) <= 1e-13 * sv[0]


def test_oracle_diagonal_band_is_fixed_point():
    S = np.diag(np.arange(1.0, 8.0))
    d, e, _ = sb2st(S, 3)
    assert np.array_equal(d, np.arange(1.0, 8.0)) or np.allclose(d, np.arange(1.0, 8.0))
    assert np.all(np.abs(e) == 0.0)


# ---- GPU ----------------------------------------------------------------------

@pytest.fixture(scope="module")
def br():
    import paper_1709_00302_b200 as m

    return m


@pytest.mark.gpu
@pytest.mark.parametrize("n,w", [(300, 32), (257, 17), (400, 64), (333, 128), (96, 5), (3, 2), (4, 3)])
def test_tridiagonal_vs_oracle(br, n, w):
    S = sym_band(n, w, 7 * n + w)
    Sp = S.copy()
    Sp[np.triu_indices(n, 1)] = np.nan  # the upper triangle is never read
    d, e = br.band_to_tridiagonal(Sp, w)
    do, eo, _ = sb2st(S, w)
    scale = np.linalg.norm(S)
    # same reflectors as the sequential oracle: d, e agree to rounding
    assert np.linalg.norm(d - do) <= 1e-12 * scale
    assert np.linalg.norm(e - eo) <= 1e-12 * scale
    ev = np.linalg.eigvalsh(S)
    assert np.max(np.abs(tri_eigs(d, e) - ev)) <= 1e-12 * np.max(np.abs(ev))


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,w", [(300, 300, 32), (310, 257, 17), (400, 400, 64), (333, 333, 128),
                                   (96, 96, 5), (3, 3, 2)])
def test_bidiagonal_vs_oracle(br, m, n, w):
    B = upper_band(m, n, w, 3 * m + n + w)
    d, e = br.band_to_bidiagonal(B, w)
    do, eo, _ = tb2bd(B, w)
    scale = np.linalg.norm(B)
    assert np.linalg.norm(d - do) <= 1e-12 * scale
    assert np.linalg.norm(e - eo) <= 1e-12 * scale
    sv = np.linalg.svd(B, compute_uv=False)
    assert np.max(np.abs(bi_svals(d, e) - sv)) <= 1e-12 * sv[0]


@pytest.mark.gpu
def test_wide_band_to_bidiagonal_transposes(br):
    """m < n: the triangular-band output of a wide matrix is a LOWER band
    (ref svd.py:221-232); it is reduced through its transpose."""
    A = np.asfortranarray(np.random.default_rng(3).standard_normal((100, 120)))
    res = br.reduce_tri_band(A, 9, 9)
    assert (res.lower_bw, res.upper_bw) == (9, 0)
    d, e = br.band_to_bidiagonal(res.band, 9)
    sv = np.linalg.svd(A, compute_uv=False)
    assert np.max(np.abs(bi_svals(d, e) - sv)) <= 1e-12 * sv[0]


_SEQ = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1709_00302_b200 as br
rng = np.random.default_rng(11)
n, w = 600, 24
g = rng.standard_normal((n, n)); S = (g + g.T) / 2
i, j = np.indices((n, n)); S[np.abs(i - j) > w] = 0
B = rng.standard_normal((n, n)); B[(j < i) | (j > i + w)] = 0
d, e = br.band_to_tridiagonal(S, w)
d2, e2 = br.band_to_bidiagonal(B, w)
np.save(sys.argv[1], np.concatenate([d, e, d2, e2]))
"""


@pytest.mark.gpu
def test_pipelined_sweeps_equal_sequential_order(tmp_path):
    """Sweeps in flight on the whole device == one sweep at a time, bitwise
    (the inter-sweep waits cover every overlapping task)."""
    outs = []
    for cap in ("0", "1"):
        f = str(tmp_path / f"r{cap}.npy")
        env = dict(os.environ, BR_S2_CTAS=cap)
        subprocess.run([sys.executable, "-c", _SEQ.format(root=ROOT), f], env=env, check=True)
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.gpu
def test_c1_c2_two_stage_pipeline(br):
    """Dense -> band (first stage) -> tridiagonal / bidiagonal (second stage)
    at the BASELINE c1 / c2 sizes: spectra of A."""
    import oracle as O

    A = O.gen_c1()
    band = br.reduce_sym_band(A, br.SevpConfig(2048, 32, 32, br.SevpVariant.V2)).band
    d, e = br.band_to_tridiagonal(band, 32)
    ev = np.linalg.eigvalsh(A)
    assert np.max(np.abs(tri_eigs(d, e) - ev)) <= 1e-10 * np.max(np.abs(ev))
    A2 = O.gen_c2()
    tb = br.reduce_tri_band(A2, 32, 32).band
    d2, e2 = br.band_to_bidiagonal(tb, 32)
    sv = np.linalg.svd(A2, compute_uv=False)
    assert np.max(np.abs(bi_svals(d2, e2) - sv)) <= 1e-10 * sv[0]


def test_stage2_rejects_wide_bands():
    import paper_1709_00302_b200 as m

    with pytest.raises(ValueError):
        m.band_to_tridiagonal(np.eye(4), 200)
    with pytest.raises(ValueError):
        m.band_to_bidiagonal(np.eye(4), 0)
