"""Multi-GPU host logic (1D block-cyclic) on CPU: two gloo
ranks run the same distributed driver as the GPUs, with NumPy stand-ins for
the rank-local kernels (test-only), and rank 0 compares the gathered band
with the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1709_00302_b200 import dist as D


class NumpyOps:
    """Rank-local dense kernels on CPU tensors (test stand-in for CudaOps)."""

    torch = torch

    def alloc(self, rows, cols, zero=False):
        return D.CMat.alloc(torch, rows, cols, torch.device("cpu"), zero=True)

    def panel_stream(self, on):
        pass

    def join(self, waiter_panel):
        pass

    def qr_panel(self, P, Y, T, W, tau, lq=False):
        A = P.numpy()
        Yn, Tn, Wn, _, tn = (O.lq_panel if lq else O.qr_panel)(A)
        Y.numpy()[...] = Yn
        T.numpy()[...] = Tn
        if W is not None:
            W.numpy()[...] = Wn
        tau.numpy()[:, 0] = tn

    def gemm(self, Cm, A, B, alpha=1.0, beta=0.0, ta=False, tb=False):
        a = A.numpy().T if ta else A.numpy()
        bb = B.numpy().T if tb else B.numpy()
        c = Cm.numpy()
        c[...] = alpha * (a @ bb) + (beta * c if beta != 0.0 else 0.0)

    def symm_acc(self, X, S, W, alpha=1.0, beta=1.0):
        s = S.numpy()
        sym = np.tril(s) + np.tril(s, -1).T
        x = X.numpy()
        x[...] = alpha * (sym @ W.numpy()) + beta * x

    def syr2k_cols(self, blk, j, cc0, X3, Y):
        a = blk.numpy()  # rows cc0..j-1 of A2, columns cc0..cc0+b
        b = a.shape[1]
        x3, y = X3.numpy(), Y.numpy()
        upd = x3[cc0:j] @ y[cc0:cc0 + b].T + y[cc0:j] @ x3[cc0:cc0 + b].T
        r = np.arange(j - cc0)[:, None]
        c = np.arange(b)[None, :]
        a[r >= c] += upd[r >= c]

    def zero(self, M):
        M.numpy()[...] = 0.0

    def copy(self, dst, src):
        dst.numpy()[...] = src.numpy()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, n, b, lookahead, out_path):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        g = rng.standard_normal((n, n))
        A = np.asfortranarray((g + g.T) / 2 if kind == "sevp" else g)
        lay = D.Layout(n, b, world, rank)
        ops = NumpyOps()
        comm = D.TorchComm(dist)
        L = D.scatter_columns(A, lay, ops)
        if kind == "sevp":
            it = D.reduce_sym_band_dist(L, lay, b, ops, comm, lookahead)
        else:
            it = D.reduce_tri_band_dist(L, lay, b, ops, comm, lookahead)
        band = D.gather_band(L, lay, b, kind, comm, torch)
        if rank == 0:
            np.savez(out_path, band=band, it=it, A=A)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,b,lookahead", [("sevp", 64, 8, 1), ("sevp", 48, 8, 0),
                                                ("tri", 64, 8, 1), ("tri", 40, 8, 0)])
def test_block_cyclic_two_ranks_matches_oracle(tmp_path, kind, n, b, lookahead):
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), kind, n, b, lookahead, out), nprocs=2, join=True)
    r = np.load(out)
    A, band = r["A"], r["band"]
    if kind == "sevp":
        ref, _, it = O.reduce_sym_band(A, n, b, b)
        assert O.band_check(band, b, b) == 0.0
        assert np.array_equal(band, band.T)
    else:
        ref, _, _, it = O.reduce_tri_band(A, b, b)
        assert O.band_check(band, 0, b) == 0.0
    assert int(r["it"]) == it
    err = np.linalg.norm(band - ref) / np.linalg.norm(A)
    assert err <= 1e-12 * np.sqrt(n), err


def test_layout_is_block_cyclic():
    lay = D.Layout(64, 8, 3, 1)
    assert lay.owned == [1, 4, 7] and lay.owner(5) == 2 and lay.slot(7) == 2
    with pytest.raises(ValueError):
        D.Layout(60, 8, 2, 0)
