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

    def flat(self, count):
        return torch.zeros(max(int(count), 1), dtype=torch.float64)

    @staticmethod
    def _map(nc, bs, r0, stride):
        c = np.arange(nc)
        return r0 + (c // bs) * stride + c % bs

    def symm_cyc(self, Xc, L, W, r0, stride, p0, p1):
        """Slab share of sym(A2) W, rows [p0, p1) (br_symm_lower_cyclic)."""
        w = W.numpy()
        nc = L.cols
        out = np.zeros((p1 - p0, w.shape[1]))
        if nc:
            l = L.numpy()
            mp = self._map(nc, w.shape[1], r0, stride)
            assert np.all(np.triu(l[mp], 1) == 0.0) and all(np.all(l[: mp[c], c] == 0.0) for c in range(nc))
            wown = w[mp]
            out += (l @ wown)[p0:p1]
            xo = l.T @ w - l[mp, np.arange(nc)][:, None] * wown
            sel = (mp >= p0) & (mp < p1)
            out[mp[sel] - p0] += xo[sel]
        Xc.numpy()[...] = out

    def syr2k_cyc(self, L, X3, Y, r0, stride):
        """Lower part of X3 Y^T + Y X3^T at the slab's columns (br_syr2k_lower_cyclic)."""
        if L.cols == 0:
            return
        l, x3, y = L.numpy(), X3.numpy(), Y.numpy()
        mp = self._map(L.cols, y.shape[1], r0, stride)
        upd = x3 @ y[mp].T + y @ x3[mp].T
        mask = np.arange(l.shape[0])[:, None] >= mp[None, :]
        l[mask] += upd[mask]

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


def _worker(rank, world, port, kind, n, b, lookahead, out_path, chunk_rows=D.CHUNK_ROWS):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        g = rng.standard_normal((n, n))
        A = np.asfortranarray((g + g.T) / 2 if kind == "sevp" else g)
        if kind == "sevp":
            A[np.triu_indices(n, 1)] = np.nan  # the upper triangle is never read
        lay = D.Layout(n, b, world, rank)
        ops = NumpyOps()
        comm = D.TorchComm(dist)
        L = D.scatter_columns(A, lay, ops, kind)
        if kind == "sevp":
            it = D.reduce_sym_band_dist(L, lay, b, ops, comm, lookahead, chunk_rows=chunk_rows)
        else:
            it = D.reduce_tri_band_dist(L, lay, b, ops, comm, lookahead, chunk_rows=chunk_rows)
        band = D.gather_band(L, lay, b, kind, comm, torch)
        if rank == 0:
            np.savez(out_path, band=band, it=it, A=A)
    finally:
        dist.destroy_process_group()


# world sizes 2, 3, 4; block counts that are not multiples of the world size
# (9 = 3 x 3 blocks over 2 or 4 ranks, 7 blocks over 3); chunk_rows = b forces
# one all-reduce chunk per block row (the pipelined path)
@pytest.mark.parametrize("world,kind,n,b,lookahead,chunk", [
    (2, "sevp", 64, 8, 1, 8192), (2, "sevp", 48, 8, 0, 8), (2, "tri", 64, 8, 1, 8192),
    (2, "tri", 40, 8, 0, 8), (3, "sevp", 56, 8, 1, 16), (3, "tri", 56, 8, 1, 8),
    (4, "sevp", 72, 8, 1, 8), (4, "tri", 72, 8, 0, 16), (4, "sevp", 72, 8, 0, 8192),
    (3, "tri", 63, 9, 1, 8192)])
def test_block_cyclic_ranks_match_oracle(tmp_path, world, kind, n, b, lookahead, chunk):
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), kind, n, b, lookahead, out, chunk), nprocs=world,
             join=True)
    r = np.load(out)
    A, band = r["A"], r["band"]
    if kind == "sevp":
        A = np.tril(A) + np.tril(A, -1).T
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
