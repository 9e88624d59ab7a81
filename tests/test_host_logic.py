"""Host-side logic of the drop-in that runs without a GPU: configs and their
validation (same errors as the reference), schedules, reference-equivalent
flop accounting, and the no-CPU-fallback rule."""
import os
import warnings

import numpy as np
import pytest

import oracle as O
import paper_1709_00302_b200 as br
from paper_1709_00302_b200 import flops as F
from paper_1709_00302_b200 import sevp as S

G = os.path.join(os.path.dirname(__file__), "golden")
RED = np.load(os.path.join(G, "reductions.npz"))

SEVP = [("s64_8_8", "reference"), ("s100_12_5", "reference"), ("s130_16_16", "v2"),
        ("s97_16_16", "reference"), ("s256_32_32", "v2"), ("s200_40_10", "v1"),
        ("s300_64_64", "reference")]
TRI = ["t64_8_8", "t100_80_12_5", "t70_90_6_6", "t256_32_32", "t97_16_16", "t300_64_64"]


@pytest.mark.parametrize("name,variant", SEVP)
def test_sevp_flops_equal_reference_counter(name, variant):
    n, w, b, iters, flops = (int(x) for x in RED[f"{name}_meta"])
    got, it = F.sevp_counted_flops(n, w, b, variant)
    assert it == iters and got["total"] == flops


@pytest.mark.parametrize("name", TRI)
def test_tri_flops_equal_reference_counter(name):
    m, n, w, b, iters, flops, _, _ = (int(x) for x in RED[f"{name}_meta"])
    got, it = F.tri_counted_flops(m, n, w, b)
    assert it == iters and got["total"] == flops


def test_counted_flops_track_nominal():
    # pkg/tests/test_sevp.py:237-241 and AC5 (5% / 8% / 10%)
    got, _ = F.sevp_counted_flops(1000, 16, 8)
    assert abs(got["total"] - F.sevp_nominal_flops(1000)) <= 0.05 * F.sevp_nominal_flops(1000)
    got, _ = F.tri_counted_flops(1000, 1000, 16, 8)
    assert abs(got["total"] - F.svd_nominal_flops(1000, 1000)) <= 0.08 * F.svd_nominal_flops(1000, 1000)


def test_nominal_flops_formulas():
    assert br.sevp_nominal_flops(0) == 0 and br.sevp_nominal_flops(3) == 36
    assert br.svd_nominal_flops(9, 9) == 1944 and br.svd_nominal_flops(12, 8) == 2389
    with pytest.raises(ValueError):
        br.sevp_nominal_flops(-1)
    with pytest.raises(ValueError):
        br.svd_nominal_flops(8, 12)


def test_schedules_match_oracle():
    for n, w, b in ((2048, 32, 32), (130, 16, 16), (97, 16, 16), (100, 12, 5), (5, 4, 2)):
        assert S._schedule(n, w, b) == O.sevp_schedule(n, w, b)


def test_config_validation_like_reference():
    # pkg/tests/test_sevp.py:207-220
    with pytest.raises(ValueError):
        br.SevpConfig(20, 4, 3, br.SevpVariant.V1).validate()
    with pytest.warns(RuntimeWarning):
        br.SevpConfig(20, 6, 2, br.SevpVariant.V2).validate()
    for bad in (br.SevpConfig(0, 2, 1), br.SevpConfig(8, 0, 1), br.SevpConfig(8, 2, 3)):
        with pytest.raises(ValueError):
            bad.validate()
    # pkg/tests/test_svd.py:302-304: triband accepts only the reference schedule
    with pytest.raises(ValueError):
        br.SvdConfig(8, 8, 2, 2, br.SvdForm.TRIANGULAR_BAND, br.SvdVariant.V2).validate()
    with pytest.raises(ValueError):
        br.SvdConfig(8, 8, 4, 3, br.SvdForm.BAND, br.SvdVariant.V1).validate()


def test_input_validation_precedes_device_work():
    """Shape / argument errors are ValueError with no GPU involved."""
    with pytest.raises(ValueError):
        br.reduce_sym_band(np.zeros((4, 5)), br.SevpConfig(4, 2, 1))
    with pytest.raises(ValueError):
        br.reduce_sym_band(np.zeros((8, 8)), br.SevpConfig(9, 2, 1))
    with pytest.raises(ValueError):
        br.reduce_sym_band(np.zeros((8, 8)), br.SevpConfig(8, 2, 3))
    with pytest.raises(ValueError):
        br.reduce_tri_band(np.zeros((8, 6)), w=0, b=1)
    with pytest.raises(ValueError):
        br.reduce_tri_band(np.zeros((8, 6)), w=2, b=3)
    with pytest.raises(ValueError):
        br.reduce_tri_band(np.zeros(5), w=2, b=1)
    with pytest.raises(ValueError):
        br.qr_panel(np.zeros((2, 3)))
    with pytest.raises(ValueError):
        br.lq_panel(np.zeros((3, 2)))
    with pytest.raises(ValueError):
        br.reduce_sym_band(np.zeros((8, 8)), br.SevpConfig(8, 2, 1), lookahead=2)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    A = np.eye(40)
    with pytest.raises(RuntimeError):
        br.reduce_sym_band(A, br.SevpConfig(40, 4, 4))
    with pytest.raises(RuntimeError):
        br.reduce_tri_band(A, 4, 4)
    with pytest.raises(RuntimeError):
        br.qr_panel(np.ones((8, 2)))


def test_band_form_not_silently_computed_on_cpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    for var in br.SvdVariant:
        with pytest.raises(RuntimeError):
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                br.reduce_band_svd(np.ones((20, 20)), br.SvdConfig(20, 20, 4, 2, variant=var))
    with pytest.raises(RuntimeError):  # wide input reduces the transpose, same path
        br.reduce_band_svd(np.ones((10, 20)), br.SvdConfig(10, 20, 4, 2))


def test_band_form_validation_matches_reference():
    with pytest.raises(ValueError, match="V1 requires 2b <= w"):
        br.reduce_band_svd(np.ones((20, 20)), br.SvdConfig(20, 20, 4, 3, variant=br.SvdVariant.V1))
    with pytest.raises(ValueError, match="need 1 <= b <= w"):
        br.reduce_band_svd(np.ones((20, 20)), br.SvdConfig(20, 20, 4, 5))
    with pytest.raises(ValueError, match="range logging is defined for the reference"):
        br.reduce_band_svd(np.ones((20, 20)),
                           br.SvdConfig(20, 20, 4, 2, variant=br.SvdVariant.SIMULTANEOUS),
                           range_log=[])
    with pytest.raises(ValueError, match="cfg says"):
        br.reduce_band_svd(np.ones((20, 21)), br.SvdConfig(20, 20, 4, 2))


def test_exec_groups_maps_to_lookahead_depth():
    assert S._depth(br.SevpConfig(8, 4, 4), br.ExecGroups(4, 0), None) == 0
    assert S._depth(br.SevpConfig(8, 4, 4, br.SevpVariant.V2), br.ExecGroups(4, 1), None) == 1
    assert S._depth(br.SevpConfig(8, 4, 4), None, None) == 0
    assert S._depth(br.SevpConfig(8, 4, 4), None, 1) == 1


def test_factor_panel_enumeration_matches_schedules():
    """The packed factor layout's panel lists (factors.py) follow the
    reference schedules (ref sevp.py:110-122, svd.py:179-202, 265-306)."""
    import oracle as O
    from paper_1709_00302_b200 import factors as F

    for n, w, b in [(100, 8, 8), (131, 12, 5), (64, 16, 16), (40, 40, 8)]:
        ks = O.sevp_schedule(n, w, b)
        p = F.sevp_panels(n, w, b)
        assert [q[0] for q in p] == ks
        assert all(q[1] == q[0] + w and q[2] == n - q[0] - w and q[3] == min(b, n - q[0] - w) for q in p)
    for m, n, w, b in [(100, 100, 8, 8), (120, 70, 10, 4), (33, 33, 16, 16)]:
        left, right = F.tri_panels(m, n, w, b)
        assert [(q[0], q[3]) for q in left] == O.tri_schedule(m, n, b)
        for k, r0, rows, cols in right:
            assert r0 == k + w and rows == n - k - w and cols == min(b, n - k, m - k, rows)
    for m, n, w, b in [(100, 100, 8, 8), (120, 70, 10, 4)]:
        left, right = F.band_panels(m, n, w, b)
        sched = O.band_schedule(m, n, w, b)
        assert [(q[0], q[3]) for q in left] == [(s[0], s[1]) for s in sched]
        assert [(q[0], q[3]) for q in right] == [(s[0], s[3]) for s in sched if s[2] >= 1]


def test_reference_driver_bounded_sample():
    """bench.py's reference arm runs the installed reference package itself on
    a bounded sample (baseline/ref_driver.py); its truncated run equals the
    oracle's first iterations."""
    import numpy as np
    import pytest

    from baseline import ref_driver as R

    if not R.available():
        pytest.skip("reference package not installed in baseline/_ref")
    import oracle as O

    mod = R.load("blas")
    A = np.asfortranarray(np.random.default_rng(3).standard_normal((96, 96)))
    fl, dt, done = R.sample(mod, "tri", A, 96, 8, 8, 3)
    assert done == 3 and fl > 0 and dt > 0
    S = (A + A.T) / 2
    fl, dt, done = R.sample(mod, "sevp", S, 96, 8, 8, 4)
    assert done == 4 and fl > 0
    # the pure (unmodified) reference and the BLAS-rebound one agree on a full run
    full_b = mod.reduce_tri_band(A, 8, 8).band
    mod = R.load("pure")
    full_p = mod.reduce_tri_band(A, 8, 8).band
    R.load("blas")
    assert np.linalg.norm(full_b - full_p) <= 1e-13 * np.linalg.norm(A)
    band, _, _, _ = O.reduce_tri_band(A, 8, 8)
    assert np.linalg.norm(full_b - band) <= 1e-13 * np.linalg.norm(A)
