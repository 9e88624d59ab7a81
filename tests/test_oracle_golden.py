"""Pin the NumPy oracle against golden vectors produced by the reference
package itself (tests/golden/make_golden.py). CPU only."""
import os

import numpy as np
import pytest

import oracle as O

G = os.path.join(os.path.dirname(__file__), "golden")
KER = np.load(os.path.join(G, "kernels.npz"))
RED = np.load(os.path.join(G, "reductions.npz"))


def rel(a, b, scale):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b))) / scale


@pytest.mark.parametrize("name", ["h345", "hzero", "hzerotail", "hneg1", "hx0zero", "hrand"])
def test_house_gen_matches_reference(name):
    v, tau, beta = O.house_gen(KER[f"{name}_x"])
    tb = KER[f"{name}_tb"]
    assert tau == tb[0] and beta == tb[1]  # bitwise: same scalar formulas
    assert np.array_equal(v, KER[f"{name}_v"])


def test_house_known_answers():
    # pkg/tests/test_kernels.py:147-181
    assert O.house_gen(np.array([3.0, 4.0]))[2] == -5.0
    v, tau, beta = O.house_gen(np.array([2.0, 0.0, 0.0]))
    assert (tau, beta) == (2.0, -2.0) and np.array_equal(v, [1.0, 0.0, 0.0])
    assert O.house_gen(np.array([-3.0]))[1:] == (2.0, 3.0)
    assert O.house_gen(np.zeros(4))[1:] == (0.0, 0.0)


QR = ["qr_40x6", "qr_sq8", "qr_257x32", "qr_300x40", "qr_tri", "qr_zerocol"]


@pytest.mark.parametrize("name", QR)
def test_qr_panel_matches_reference(name):
    P = KER[f"{name}_in"].copy(order="F")
    Y, T, W, R, tau = O.qr_panel(P)
    s = np.linalg.norm(KER[f"{name}_in"]) + 1.0
    assert np.array_equal(np.sign(np.diag(R)), np.sign(np.diag(KER[f"{name}_R"])))
    for got, key in ((Y, "Y"), (T, "T"), (W, "W"), (R, "R"), (tau, "tau"), (P, "out")):
        ref = KER[f"{name}_{key}"]
        assert rel(got, ref, max(1.0, np.linalg.norm(ref))) <= 1e-13, key
    assert rel(R, KER[f"{name}_R"], s) <= 1e-14


@pytest.mark.parametrize("name", ["lq_6x40", "lq_32x257", "lq_sq8"])
def test_lq_panel_matches_reference(name):
    P = KER[f"{name}_in"].copy(order="F")
    Y, T, W, L, tau = O.lq_panel(P)
    for got, key in ((Y, "Y"), (T, "T"), (W, "W"), (L, "L"), (tau, "tau"), (P, "out")):
        ref = KER[f"{name}_{key}"]
        assert rel(got, ref, max(1.0, np.linalg.norm(ref))) <= 1e-13, key


def test_wy_apply_matches_reference():
    A = KER["awl_in"].copy(order="F")
    O.apply_wy_left(A, KER["awl_Y"], KER["awl_W"])
    assert rel(A, KER["awl_out"], np.linalg.norm(KER["awl_in"])) <= 1e-14
    A = KER["awr_in"].copy(order="F")
    O.apply_wy_right(A, KER["awr_Y"], KER["awr_W"])
    assert rel(A, KER["awr_out"], np.linalg.norm(KER["awr_in"])) <= 1e-14


def test_symmetric_kernels_match_reference():
    X1 = O.symm_lower(KER["symm_A"], KER["symm_W"])
    assert rel(X1, KER["symm_X1"], np.linalg.norm(KER["symm_X1"])) <= 1e-14
    S = KER["syr_A"].copy(order="F")
    O.syr2k_lower(S, KER["syr_X3"], KER["syr_Y"], 0, S.shape[0])
    assert np.array_equal(np.triu(S, 1), np.triu(KER["syr_out"], 1))  # upper untouched
    assert rel(np.tril(S), np.tril(KER["syr_out"]), np.linalg.norm(np.tril(KER["syr_out"]))) <= 1e-14
    S = KER["syr_A"].copy(order="F")
    O.syr2k_lower(S, KER["syr_X3"], KER["syr_Y"], 37, 101)
    assert np.array_equal(np.triu(S, 1), np.triu(KER["syr_part_out"], 1))
    assert rel(np.tril(S), np.tril(KER["syr_part_out"]), np.linalg.norm(np.tril(S))) <= 1e-14
    S = KER["tsu_A"].copy(order="F")
    O.sym_two_sided_update(S, KER["tsu_Y"], KER["tsu_W"])
    assert rel(np.tril(S), np.tril(KER["tsu_out"]), np.linalg.norm(np.tril(S))) <= 1e-13


SEVP = ["s64_8_8", "s100_12_5", "s130_16_16", "s97_16_16", "s256_32_32", "s200_40_10", "s300_64_64"]


@pytest.mark.parametrize("name", SEVP)
def test_reduce_sym_band_matches_reference(name):
    n, w, b, iters, _ = RED[f"{name}_meta"]
    A = RED[f"{name}_A"]
    band, _, it = O.reduce_sym_band(A, int(n), int(w), int(b))
    assert it == iters
    assert O.band_check(band, w, w) == 0.0
    assert np.array_equal(band, band.T)
    scale = np.linalg.norm(np.tril(A) + np.tril(A, -1).T)
    assert rel(band, RED[f"{name}_band"], scale) <= 1e-12 * np.sqrt(n)
    assert rel(band, RED[f"{name}_band"], scale) <= 1e-13


def test_reduce_sym_band_q_matches_reference():
    band, Q, _ = O.reduce_sym_band(RED["sq_A"], 48, 6, 3, accumulate_q=True)
    assert rel(band, RED["sq_band"], np.linalg.norm(RED["sq_A"])) <= 1e-13
    assert rel(Q, RED["sq_Q"], 1.0) <= 1e-13


TRI = ["t64_8_8", "t100_80_12_5", "t70_90_6_6", "t256_32_32", "t97_16_16", "t300_64_64"]


@pytest.mark.parametrize("name", TRI)
def test_reduce_tri_band_matches_reference(name):
    m, n, w, b, iters, _, lbw, ubw = RED[f"{name}_meta"]
    A = RED[f"{name}_A"]
    band, lo, up, it = O.reduce_tri_band(A, int(w), int(b))
    assert (lo, up, it) == (lbw, ubw, iters)
    assert O.band_check(band, lo, up) == 0.0
    scale = np.linalg.norm(A)
    assert rel(band, RED[f"{name}_band"], scale) <= 1e-13


def test_nominal_flops():
    # pkg/tests/test_sevp.py:230-234, pkg/tests/test_svd.py:315-320
    assert O.sevp_nominal_flops(3) == 36
    assert O.svd_nominal_flops(9, 9) == 1944
    assert O.svd_nominal_flops(12, 8) == 2389


BAND = np.load(os.path.join(G, "band.npz"))
BAND_CASES = sorted({k[: -len("_meta")] for k in BAND.files if k.endswith("_meta")})


@pytest.mark.parametrize("name", BAND_CASES)
def test_reduce_band_svd_matches_reference(name):
    m, n, w, b, iters, flops, lbw, ubw = (int(x) for x in BAND[f"{name}_meta"])
    A = BAND[f"{name}_A"]
    sim = name.endswith(("_sim", "_v2"))
    band, lo, up, it = O.reduce_band_svd(A, w, b, simultaneous=sim)
    assert (lo, up, it) == (lbw, ubw, iters)
    assert O.band_check(band, lo, up) == 0.0
    assert rel(band, BAND[f"{name}_band"], np.linalg.norm(A)) <= 1e-13


@pytest.mark.parametrize("name", BAND_CASES)
def test_band_counted_flops_match_reference(name):
    from paper_1709_00302_b200.flops import band_counted_flops

    m, n, w, b, iters, flops, _, _ = (int(x) for x in BAND[f"{name}_meta"])
    got, it = band_counted_flops(m, n, w, b, simultaneous=name.endswith(("_sim", "_v2")))
    assert (got["total"], it) == (flops, iters)


def test_band_form_small_input_unchanged():
    # m <= w + 1: nothing is off-band (ref svd.py:561-564)
    A = np.random.default_rng(3).standard_normal((5, 5))
    band, lo, up, it = O.reduce_band_svd(A, 4, 2)
    assert it == 0 and np.array_equal(band, A) and (lo, up) == (4, 4)
