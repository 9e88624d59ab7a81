"""Returned Householder factors (`return_factors=True`, C-ABI `br_factors`)
and the north-star backward error.

The reference keeps every panel's factors in private state
(ref sevp.py:128-134 state.factors[k]; ref svd.py:185,195 fu / fv); the
oracle restates that (its `factors=` hook). Checked here:
  * each panel's Y, T, tau against the oracle's (<= 1e-12 relative, the
    band-parity bound; the sign conventions make them unique);
  * Q (SEVP) / U, V (SVD) formed from the factors on the GPU are orthogonal
    and reproduce A: ||A - Q B Q^T||_F / (n eps ||A||_F) = O(1) (north_star's
    backward-error criterion; asserted <= 10), and Q equals accumulate_q's;
  * the reference's own SEVP check ||Q^T A Q - B||_F <= 1e-12 ||A||_F
    (pkg/tests/test_sevp.py:67-72).
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def br():
    import paper_1709_00302_b200 as m

    return m


def sym(n, seed):
    g = np.random.default_rng(seed).standard_normal((n, n))
    return np.asfortranarray((g + g.T) / 2.0)


def rand(m, n, seed):
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((m, n)))


def backward_error(A, L, B, R):
    """||A - L B R^T||_F / (max(m, n) eps ||A||_F)."""
    return np.linalg.norm(A - L @ B @ R.T) / (max(A.shape) * EPS * np.linalg.norm(A))


def orth(Q):
    return np.linalg.norm(Q.T @ Q - np.eye(Q.shape[1])) / (Q.shape[0] * EPS)


def close(a, b, tol=1e-12):
    return np.linalg.norm(a - b) <= tol * max(1.0, np.linalg.norm(b))


@pytest.mark.parametrize("n,w,b,variant", [(200, 16, 16, "V2"), (230, 24, 8, "V1"), (97, 12, 12, "REFERENCE"),
                                           (129, 16, 16, "V2")])
def test_sevp_factors_vs_oracle_and_backward_error(br, n, w, b, variant):
    A = sym(n, n)
    cfg = br.SevpConfig(n, w, b, getattr(br.SevpVariant, variant), accumulate_q=True)
    res = br.reduce_sym_band(A, cfg, return_factors=True)
    ref = {}
    band, _, _ = O.reduce_sym_band(A, n, w, b, factors=ref)
    assert np.linalg.norm(res.band - band) <= 1e-12 * np.sqrt(n) * np.linalg.norm(A)
    f = res.factors.left
    assert sorted(f.keys()) == sorted(ref.keys()) and res.factors.right is None
    for k, (Y, T, tau) in ref.items():
        p = f[k]
        assert close(p.y, Y) and close(p.t, T) and close(p.tau, tau), k
        assert np.array_equal(np.diag(p.y), np.ones(p.y.shape[1]))  # unit diagonal, exact
        assert np.all(np.triu(p.y, 1) == 0.0)
    Q = f.form_q()
    assert orth(Q) <= 10.0
    assert np.linalg.norm(Q - res.q) <= 1e-12 * n  # the same product as accumulate_q
    assert backward_error(A, Q, res.band, Q) <= 10.0
    # pkg/tests/test_sevp.py:67-72
    assert np.linalg.norm(Q.T @ A @ Q - res.band) <= 1e-12 * np.linalg.norm(A)


@pytest.mark.parametrize("m,n,w,b", [(200, 200, 16, 16), (300, 170, 20, 10), (150, 150, 32, 8),
                                     (65, 65, 16, 16)])
def test_tri_factors_vs_oracle_and_backward_error(br, m, n, w, b):
    A = rand(m, n, m + n)
    res = br.reduce_tri_band(A, w, b, return_factors=True)
    ref = {}
    band, _, _, _ = O.reduce_tri_band(A, w, b, factors=ref)
    assert np.linalg.norm(res.band - band) <= 1e-12 * np.sqrt(n) * np.linalg.norm(A)
    U, V = res.factors.left, res.factors.right
    assert sorted(U.keys()) == sorted(k for c, k in ref if c == "qr")
    assert sorted(V.keys()) == sorted(k for c, k in ref if c == "lq")
    for (c, k), (Y, T, tau) in ref.items():
        p = (U if c == "qr" else V)[k]
        assert close(p.y, Y) and close(p.t, T) and close(p.tau, tau), (c, k)
    Uq, Vq = U.form_q(), V.form_q()
    assert Uq.shape == (m, m) and Vq.shape == (n, n)
    assert orth(Uq) <= 10.0 and orth(Vq) <= 10.0
    assert backward_error(A, Uq, res.band, Vq) <= 10.0


def test_tri_factors_wide_matrix(br):
    # m < n: the transpose is reduced; A = U B V^T still holds with the chains swapped
    A = rand(90, 160, 7)
    res = br.reduce_tri_band(A, 12, 6, return_factors=True)
    U, V = res.factors.left.form_q(), res.factors.right.form_q()
    assert U.shape == (90, 90) and V.shape == (160, 160)
    assert backward_error(A, U, res.band, V) <= 10.0


@pytest.mark.parametrize("variant", ["REFERENCE", "SIMULTANEOUS", "V1", "V2"])
def test_band_form_factors_backward_error(br, variant):
    m, n, w = 260, 200, 24
    b = 12 if variant == "V1" else 16
    A = rand(m, n, 3)
    cfg = br.SvdConfig(m, n, w, b, br.SvdForm.BAND, getattr(br.SvdVariant, variant))
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        res = br.reduce_band_svd(A, cfg, return_factors=True)
    U, V = res.factors.left.form_q(), res.factors.right.form_q()
    assert orth(U) <= 10.0 and orth(V) <= 10.0
    assert backward_error(A, U, res.band, V) <= 10.0


def test_factors_do_not_change_the_band(br):
    A = rand(180, 180, 11)
    a = br.reduce_tri_band(A, 16, 16)
    f = br.reduce_tri_band(A, 16, 16, return_factors=True)
    assert np.array_equal(a.band, f.band)
    S = sym(180, 12)
    cfg = br.SevpConfig(180, 16, 16, br.SevpVariant.V2)
    assert np.array_equal(br.reduce_sym_band(S, cfg).band,
                          br.reduce_sym_band(S, cfg, return_factors=True).band)


def test_first_panel_factors_equal_qr_panel(br):
    # the first panel is the untouched input columns: its factors are qr_panel's
    A = rand(400, 400, 21)
    res = br.reduce_tri_band(A, 32, 32, return_factors=True)
    Y, T, W, R, tau = O.qr_panel(np.asfortranarray(A[:, :32].copy()))
    p = res.factors.left[0]
    assert close(p.y, Y) and close(p.t, T) and close(p.tau, tau) and close(p.w, W)


def test_c2_full_size_backward_error(br):
    A = O.gen_c2()
    res = br.reduce_tri_band(A, 32, 32, return_factors=True)
    U, V = res.factors.left.form_q(), res.factors.right.form_q()
    be = backward_error(A, U, res.band, V)
    print(f"c2 backward error {be:.3f}")
    assert be <= 10.0
