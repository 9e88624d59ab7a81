"""The 1D block-cyclic distributed driver on a real GPU with NCCL (world size
1 on the single test GPU: exercises the CUDA rank-local kernels - including
the block-column SYR2K/SYMM/GEMM views - and the NCCL plumbing; the
multi-rank logic itself is covered by tests/test_dist_gloo.py)."""
import socket

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl():
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,b,la", [("sevp", 512, 32, 1), ("sevp", 384, 64, 0),
                                         ("tri", 512, 32, 1), ("tri", 384, 64, 0)])
def test_distributed_driver_on_gpu(nccl, kind, n, b, la):
    import torch

    from paper_1709_00302_b200 import dist as D

    rng = np.random.default_rng(11)
    g = rng.standard_normal((n, n))
    A = np.asfortranarray((g + g.T) / 2 if kind == "sevp" else g)
    lay = D.Layout(n, b, 1, 0)
    ops = D.CudaOps(0, torch)
    comm = D.TorchComm(nccl, stream=torch.cuda.Stream())
    L = D.scatter_columns(A, lay, ops, kind)
    if kind == "sevp":
        it = D.reduce_sym_band_dist(L, lay, b, ops, comm, la, chunk_rows=2 * b)
        ref, _, it_ref = O.reduce_sym_band(A, n, b, b)
    else:
        it = D.reduce_tri_band_dist(L, lay, b, ops, comm, la)
        ref, _, _, it_ref = O.reduce_tri_band(A, b, b)
    ops.sync()
    band = D.gather_band(L, lay, b, kind, comm, torch)
    assert it == it_ref
    assert O.band_check(band, b if kind == "sevp" else 0, b) == 0.0
    assert np.linalg.norm(band - ref) / np.linalg.norm(A) <= 1e-12 * np.sqrt(n)


@pytest.mark.parametrize("world,rank,j,b", [(2, 1, 768, 64), (3, 0, 960, 64), (4, 2, 1024, 32),
                                            (3, 2, 576, 32), (1, 0, 512, 64)])
def test_cyclic_slab_kernels_vs_numpy(world, rank, j, b):
    """br_symm_lower_cyclic / br_syr2k_lower_cyclic for one rank of a
    block-cyclic partition of a j x j trailing matrix, against NumPy; the
    shares of all ranks sum to sym(A2) W."""
    import torch

    from paper_1709_00302_b200 import _lib
    from paper_1709_00302_b200 import dist as D

    lib = _lib.load()
    h = _lib.handle(0)
    lib.br_set_streams(h, None, None)
    rng = np.random.default_rng(world * 10 + rank)
    g = rng.standard_normal((j, j))
    S = (g + g.T) / 2
    Wn = rng.standard_normal((j, b))
    X3n, Yn = rng.standard_normal((j, b)), rng.standard_normal((j, b))
    nblk = j // b
    total = np.zeros((j, b))
    for r in range(world):
        blocks = [q for q in range(nblk) if q % world == r]
        cols = np.concatenate([np.arange(q * b, (q + 1) * b) for q in blocks]) if blocks else np.zeros(0, int)
        Ln = np.tril(S)[:, cols].copy()  # zero above the diagonal
        nc = len(cols)
        r0 = blocks[0] * b if blocks else 0
        ld = (j + 31) // 32 * 32
        Ld = torch.zeros((max(nc, 1), ld), dtype=torch.float64, device="cuda")
        if nc:
            Ld[:nc, :j] = torch.from_numpy(Ln.T.copy())
        Wd = torch.from_numpy(Wn.T.copy()).cuda()
        X1d = torch.full((b, j), np.nan, dtype=torch.float64, device="cuda")
        # two row chunks (on a block boundary) and the whole range
        half = (nblk // 2) * b
        for p0, p1 in ((0, half), (half, j)):
            Xc = torch.empty((b, p1 - p0), dtype=torch.float64, device="cuda")
            _lib.check(lib.br_symm_lower_cyclic(h, j, nc, b, Ld.data_ptr() if nc else None, ld,
                                                Wd.data_ptr(), j, Xc.data_ptr(), p1 - p0, r0, b,
                                                world * b, p0, p1), "symm_cyclic")
            _lib.check(lib.br_sync(h), "sync")  # the library's own stream, then torch's copy
            X1d[:, p0:p1] = Xc
        torch.cuda.synchronize()
        share = X1d.cpu().numpy().T
        ref = np.tril(S)[:, cols] @ Wn[cols] if nc else np.zeros((j, b))
        if nc:
            Lc = np.tril(S)[:, cols]
            xo = Lc.T @ Wn - np.diag(S)[cols][:, None] * Wn[cols]
            ref[cols] += xo
        assert np.linalg.norm(share - ref) <= 1e-12 * np.linalg.norm(ref) + 1e-300
        total += share
        if r == rank and nc:
            X3d = torch.from_numpy(X3n.T.copy()).cuda()
            Yd = torch.from_numpy(Yn.T.copy()).cuda()
            _lib.check(lib.br_syr2k_lower_cyclic(h, j, nc, b, Ld.data_ptr(), ld, X3d.data_ptr(), j,
                                                 Yd.data_ptr(), j, r0, b, world * b), "syr2k_cyclic")
            torch.cuda.synchronize()
            got = Ld[:nc, :j].cpu().numpy().T
            upd = X3n @ Yn[cols].T + Yn @ X3n[cols].T
            mask = np.arange(j)[:, None] >= cols[None, :]
            want = Ln + np.where(mask, upd, 0.0)
            assert np.array_equal(got[~mask], np.zeros(int((~mask).sum())))  # upper stays zero
            assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)
    sym = np.tril(S) + np.tril(S, -1).T
    assert np.linalg.norm(total - sym @ Wn) <= 1e-12 * np.linalg.norm(sym @ Wn)
