"""BASELINE.json configurations at full size on the GPU: c3 against the
oracle, and size-independent properties for c3-c5 (exact band pattern and
symmetry, Frobenius norm and trace preserved by the orthogonal two-sided
transforms, look-ahead bitwise equal to the sequential schedule, run-to-run
determinism)."""
import ctypes as C

import numpy as np
import pytest

import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _run(kind, A, w, b, la, h, lib, torch):
    from paper_1709_00302_b200 import _lib

    n = A.shape[0]
    ld = (n + 31) // 32 * 32
    d = torch.empty((n, ld), dtype=torch.float64, device="cuda")
    d[:, :n].copy_(torch.from_numpy(np.asfortranarray(A).T))
    st = _lib.BrStats()
    if kind == "sevp":
        rc = lib.br_reduce_sym_band(h, n, w, b, la, d.data_ptr(), ld, None, 0, st)
    else:
        rc = lib.br_reduce_tri_band(h, n, n, w, b, la, d.data_ptr(), ld, st)
    _lib.check(rc, "reduce")
    return d, st


@pytest.fixture(scope="module")
def env():
    import torch

    from paper_1709_00302_b200 import _lib

    lib = _lib.load()
    h = _lib.handle(0)
    lib.br_set_streams(h, None, None)
    return torch, lib, h


def test_c3_full_vs_oracle(env):
    torch, lib, h = env
    A = O.gen_c3()
    d, st = _run("sevp", A, 128, 128, 1, h, lib, torch)
    band = d[:, :8192].cpu().numpy().T
    ref, _, it = O.reduce_sym_band(A, 8192, 128, 128)
    assert st.iterations == it
    assert O.band_check(band, 128, 128) == 0.0
    assert np.linalg.norm(band - ref) / np.linalg.norm(A) <= 1e-12 * np.sqrt(8192)
    ev_a = np.linalg.eigvalsh(A)
    ev_b = torch.linalg.eigvalsh(torch.from_numpy(band).cuda()).cpu().numpy()
    assert np.max(np.abs(ev_a - ev_b)) <= 1e-10 * np.max(np.abs(ev_a))


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_large_configs_properties(env, cfg):
    torch, lib, h = env
    kind, n, w, b = {"c4": ("tri", 16384, 256, 256), "c5": ("sevp", 32768, 256, 256)}[cfg]
    A = O.gen_config(cfg)
    nA = float(np.linalg.norm(A))  # c5's generator is exactly symmetric
    trA = float(np.trace(A))
    d1, st = _run(kind, A, w, b, 1, h, lib, torch)
    band = d1[:, :n]  # row-major view of the column-major band: band^T
    # exact zeros off the band, on the device
    i = torch.arange(n, device="cuda")
    r = i[None, :]  # row index of element (c, r) of the transposed view
    c = i[:, None]
    off = ((r - c) > (w if kind == "sevp" else 0)) | ((c - r) > w)
    assert float(band[off].abs().max()) == 0.0
    if kind == "sevp":
        assert torch.equal(band, band.T)
        assert abs(float(torch.trace(band)) - trA) <= 1e-10 * nA
    fro = float(torch.linalg.norm(band))
    assert abs(fro - nA) <= 1e-12 * np.sqrt(n) * nA
    del off, r, c, i
    # depth 1 == depth 0 bitwise, and run-to-run determinism
    d0, _ = _run(kind, A, w, b, 0, h, lib, torch)
    assert torch.equal(d0[:, :n], band)
    del d0
    d2, _ = _run(kind, A, w, b, 1, h, lib, torch)
    assert torch.equal(d2[:, :n], band)
