"""Single-process multi-device driver (multi.py, the `ngpus` / `devices`
extension of SURVEY.md 8(b)) on CPU: rank THREADS run the block-cyclic
driver with NumPy stand-ins for the rank-local kernels (test-only) and the
host rendezvous collectives; rank 0's band must equal the single-process
oracle, and the per-panel taus must not depend on the rank count."""
import threading

import numpy as np
import pytest

import oracle as O
from paper_1709_00302_b200 import multi as M
from test_dist_gloo import NumpyOps


def _input(kind, n, seed=11):
    g = np.random.default_rng(seed).standard_normal((n, n))
    A = np.asfortranarray((g + g.T) / 2 if kind == "sevp" else g)
    return A


def _run(A, kind, b, world, lookahead, chunk=M.D.CHUNK_ROWS):
    return M.reduce_on_ranks(A, kind, b, b, world, lambda r: NumpyOps(), M.HostGroup(world),
                             lookahead, chunk_rows=chunk)


@pytest.mark.parametrize("world,kind,n,b,lookahead,chunk", [
    (1, "sevp", 48, 8, 1, 8192), (2, "sevp", 64, 8, 1, 8), (3, "sevp", 72, 8, 0, 16),
    (4, "sevp", 72, 8, 1, 8192), (1, "tri", 40, 8, 1, 8192), (2, "tri", 64, 8, 0, 8),
    (3, "tri", 63, 9, 1, 8192), (4, "tri", 72, 8, 1, 16)])
def test_rank_threads_match_oracle(world, kind, n, b, lookahead, chunk):
    A = _input(kind, n)
    Ain = A.copy()
    if kind == "sevp":
        Ain[np.triu_indices(n, 1)] = np.nan  # the upper triangle is never read
    band, its, (taul, taur) = _run(Ain, kind, b, world, lookahead, chunk)
    if kind == "sevp":
        ref, _, it = O.reduce_sym_band(A, n, b, b)
        assert O.band_check(band, b, b) == 0.0 and np.array_equal(band, band.T)
        assert taur is None
    else:
        ref, _, _, it = O.reduce_tri_band(A, b, b)
        assert O.band_check(band, 0, b) == 0.0
    assert its == it
    err = np.linalg.norm(band - ref) / np.linalg.norm(A)
    assert err <= 1e-12 * np.sqrt(n), err
    # every panel's taus were recorded at its leading column
    npan = n - b if kind == "sevp" else n
    assert np.all(taul[:npan] != 0.0) and np.all(taul[npan:] == 0.0)
    if kind == "tri":
        assert np.all(taur[: n - b] != 0.0) and np.all(taur[n - b:] == 0.0)


def test_taus_agree_across_rank_counts():
    A = _input("tri", 48, seed=3)
    _, _, t1 = _run(A, "tri", 8, 1, 1)
    _, _, t3 = _run(A, "tri", 8, 3, 1)
    # (the all-reduced products sum in a rank-count dependent order: not bitwise)
    assert np.allclose(t1[0], t3[0], rtol=1e-12, atol=0) and np.allclose(t1[1], t3[1], rtol=1e-12, atol=0)
    assert np.array_equal(t1[0] == 0.0, t3[0] == 0.0)


def test_zero_column_tau_zero_reaches_flop_correction():
    # a matrix whose first column below the diagonal is zero: the first SEVP
    # panel has a tau == 0 reflector on rank 0, and the gathered taus carry it
    n, b = 32, 8
    A = _input("sevp", n, seed=5)
    A[b:, 0] = 0.0
    A[0, b:] = 0.0
    _, _, (taul, _) = _run(A, "sevp", b, 2, 1)
    assert taul[0] == 0.0 and np.all(taul[1:n - b] != 0.0)


class _FailingOps(NumpyOps):
    def __init__(self, rank):
        self.rank = rank

    def gemm(self, *a, **k):
        if self.rank == 1:
            raise RuntimeError("injected failure on rank 1")
        return super().gemm(*a, **k)


def test_failure_on_one_rank_raises_without_hanging():
    A = _input("tri", 32)
    before = threading.active_count()
    with pytest.raises(RuntimeError, match="injected failure"):
        M.reduce_on_ranks(A, "tri", 8, 8, 3, lambda r: _FailingOps(r), M.HostGroup(3), 1)
    assert threading.active_count() == before


def test_resolve_devices():
    assert M.resolve_devices(None, None) is None
    assert M.resolve_devices(1, None) is None  # one GPU: the native single-GPU path
    assert M.resolve_devices(4, None) == [0, 1, 2, 3]
    assert M.resolve_devices(None, [2]) == [2]  # explicit list: the driver, even on one device
    assert M.resolve_devices(2, [3, 5]) == [3, 5]
    for bad in [(0, None), (None, []), (None, [1, 1]), (3, [0, 1])]:
        with pytest.raises(ValueError):
            M.resolve_devices(*bad)


def test_public_api_rejects_unsupported_multi_gpu_shapes():
    import paper_1709_00302_b200 as br

    A = _input("sevp", 64)
    with pytest.raises(ValueError, match="w == b"):
        br.reduce_sym_band(A, br.SevpConfig(64, 16, 8), devices=[0])
    with pytest.raises(ValueError, match="multiple of b"):
        br.reduce_sym_band(A[:60, :60], br.SevpConfig(60, 8, 8), devices=[0])
    with pytest.raises(ValueError, match="single-GPU"):
        br.reduce_sym_band(A, br.SevpConfig(64, 8, 8, accumulate_q=True), ngpus=2)
    with pytest.raises(ValueError, match="square"):
        br.reduce_tri_band(A[:, :48], 8, 8, devices=[0])
    cfg = br.SvdConfig(64, 64, 8, 8, form=br.SvdForm.BAND)
    with pytest.raises(ValueError, match="band form"):
        br.reduce_band_svd(A, cfg, ngpus=2)
