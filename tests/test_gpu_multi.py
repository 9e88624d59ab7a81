"""The single-call multi-GPU path (`devices=` / `ngpus=`, multi.py) on the GPU:
rank threads drive the sm_100a library over the C ABI with single-process
NCCL collectives. On the one test GPU this runs the block-cyclic driver at
one rank (devices=[0]); with more visible GPUs it also runs every one of
them. Bands are compared with the oracle and with the native single-GPU
path; result.flops must equal the native path's (the reference's count)."""
import numpy as np
import pytest

import oracle as O
import paper_1709_00302_b200 as br

pytestmark = pytest.mark.gpu


def _devices():
    import torch

    n = torch.cuda.device_count()
    return [[0]] + ([list(range(n))] if n > 1 else [])


@pytest.mark.parametrize("n,b,la", [(512, 32, 1), (384, 64, 0), (1024, 64, 1)])
def test_sym_band_devices_matches_oracle_and_native(n, b, la):
    g = np.random.default_rng(21).standard_normal((n, n))
    A = np.asfortranarray((g + g.T) / 2)
    A_nan = A.copy()
    A_nan[np.triu_indices(n, 1)] = np.nan  # never read
    cfg = br.SevpConfig(n, b, b, br.SevpVariant.V2 if la else br.SevpVariant.REFERENCE)
    native = br.reduce_sym_band(A, cfg)
    ref, _, it = O.reduce_sym_band(A, n, b, b)
    for devs in _devices():
        res = br.reduce_sym_band(A_nan, cfg, devices=devs, lookahead=la)
        assert res.iterations == it == native.iterations
        assert br.band_check(res.band, b, b) == 0.0 and np.array_equal(res.band, res.band.T)
        for other in (ref, native.band):
            err = np.linalg.norm(res.band - other) / np.linalg.norm(A)
            assert err <= 1e-12 * np.sqrt(n), (devs, err)
        assert res.flops == native.flops


@pytest.mark.parametrize("n,b,la", [(512, 32, 1), (384, 64, 0), (1024, 64, 1)])
def test_tri_band_devices_matches_oracle_and_native(n, b, la):
    A = np.asfortranarray(np.random.default_rng(22).standard_normal((n, n)))
    native = br.reduce_tri_band(A, b, b)
    ref, _, _, it = O.reduce_tri_band(A, b, b)
    for devs in _devices():
        res = br.reduce_tri_band(A, b, b, devices=devs, lookahead=la)
        assert res.iterations == it == native.iterations
        assert br.band_check(res.band, 0, b) == 0.0
        for other in (ref, native.band):
            err = np.linalg.norm(res.band - other) / np.linalg.norm(A)
            assert err <= 1e-12 * np.sqrt(n), (devs, err)
        assert res.flops == native.flops


def test_zero_column_flops_match_native():
    # tau == 0 reflectors: the gathered per-panel taus drive the reference's
    # exact flop count on the multi-GPU path too
    n, b = 256, 32
    A = np.diag(np.arange(1.0, n + 1))
    A[40:, 3] = A[3, 40:] = 0.5
    cfg = br.SevpConfig(n, b, b, br.SevpVariant.V2)
    native = br.reduce_sym_band(A, cfg)
    res = br.reduce_sym_band(A, cfg, devices=[0])
    assert res.flops == native.flops
    # columns that are zero up to rounding noise make the later reflectors (and
    # so the band entries) depend on that noise: the bands are compared through
    # their spectra, which every valid reduction shares with A
    ev = np.linalg.eigvalsh(A)
    for band in (res.band, native.band):
        assert br.band_check(band, b, b) == 0.0
        assert np.max(np.abs(np.linalg.eigvalsh(band) - ev)) <= 1e-12 * np.max(np.abs(ev))


def test_native_path_unchanged_after_multi_call():
    # the multi runner borrows the device handle's streams and must give them back
    n, b = 256, 32
    A = np.asfortranarray(np.random.default_rng(3).standard_normal((n, n)))
    before = br.reduce_tri_band(A, b, b).band
    br.reduce_tri_band(A, b, b, devices=[0])
    after = br.reduce_tri_band(A, b, b).band
    assert np.array_equal(before, after)
