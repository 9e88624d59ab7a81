"""Multi-GPU first-stage reduction: 1D block-cyclic columns.

One process per GPU (torchrun). Block column t (width b) of the n x n matrix
lives on rank t mod P, stored locally as a column-major n x (b * #owned)
array. Per iteration k = t*b (w == b, the sharded BASELINE configs):

SEVP (ref sevp.py:194-273, look-ahead depth 1 as V2):
  1. the owner of block t factors the panel A[k+b:n, block t] (cluster leaf
     kernels) and NCCL-broadcasts Y and T; every rank forms W = Y T;
  2. every rank accumulates its owned block columns' share of
     X1 = sym(A2) W from lower-stored data only - for block c:
     X1[c] += sym(A2[c,c]) W[c];  X1[c+1:] += A2[c+1:,c] W[c];
     X1[c] += A2[c+1:,c]^T W[c+1:] - then all-reduces X1 (the distributed
     A V product, the path's real exchange step);
  3. X2 = X1^T W / 2, X3 = X1 + Y X2 on every rank (replicated, small);
  4. SYR2K on the owned block columns; look-ahead: the owner of block t+1
     updates that block first and factors the next panel on its panel
     stream while it finishes the rest.
Triangular band (ref svd.py:179-202):
  1. QR owner factors A[k:m, block t], broadcast Y_U, T_U;
  2. the left update is local to each owned block column;
  3. the LQ row panel A[k:k+b, k+b:n] spans all owners: NCCL all-gather of
     the owned b x b pieces, then every rank factors the same LQ (identical
     inputs and kernels -> bit-identical factors, no broadcast needed);
  4. right update: partial Z = D[:, owned] W_V[owned] on every rank,
     all-reduce(Z), then D[:, owned] += Z Y_V[owned]^T locally;
  5. look-ahead: block t+1's owner updates it first and factors QR(t+1) on
     its panel stream.

The algorithm is written once against two small interfaces so its host
logic is testable on CPU: `ops` (rank-local dense kernels; `CudaOps` here
drives the sm_100a library through the C ABI) and `comm` (torch.distributed:
NCCL for GPUs; the gloo tests plug NumPy ops into the same driver).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass
class Layout:
    """1D block-cyclic column map: block t -> rank t % world, slot t // world."""

    n: int
    b: int
    world: int
    rank: int

    def __post_init__(self):
        if self.n % self.b:
            raise ValueError("the distributed path needs n to be a multiple of b")
        self.nblk = self.n // self.b
        self.owned = [t for t in range(self.nblk) if t % self.world == self.rank]

    def owner(self, t: int) -> int:
        return t % self.world

    def slot(self, t: int) -> int:
        return t // self.world

    @property
    def ncols_local(self) -> int:
        return len(self.owned) * self.b


class CMat:
    """Column-major fp64 matrix on a torch tensor of shape (cols, ld)."""

    __slots__ = ("t", "rows", "cols", "ld")

    def __init__(self, t, rows, cols):
        self.t = t
        self.rows = int(rows)
        self.cols = int(cols)
        self.ld = int(t.stride(0)) if t.dim() == 2 and t.shape[0] > 1 else int(t.shape[-1])

    @classmethod
    def alloc(cls, torch, rows, cols, device, zero=False):
        ld = max(32, (rows + 31) // 32 * 32)
        f = torch.zeros if zero else torch.empty
        t = f((max(cols, 1), ld), dtype=torch.float64, device=device)
        m = cls(t, rows, cols)
        m.ld = ld
        return m

    def view(self, r0, r1, c0, c1):
        m = CMat(self.t[c0:c1, r0:r1], r1 - r0, c1 - c0)
        m.ld = self.ld
        return m

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def numpy(self):
        """(rows x cols) F-order NumPy view (CPU tensors only)."""
        return self.t[: self.cols, : self.rows].numpy().T


class CudaOps:
    """Rank-local kernels on the sm_100a library (C ABI), on the handle's
    main / panel streams; the main stream is torch's current stream so NCCL
    collectives issued by torch.distributed are ordered with the kernels."""

    def __init__(self, device: int, torch):
        self.torch = torch
        self.lib = _lib.load()
        self.h = _lib.handle(device)
        self.dev = torch.device("cuda", device)
        self.stream = torch.cuda.current_stream(self.dev)
        if self.stream.cuda_stream == 0:
            self.stream = torch.cuda.Stream(device=self.dev)
            torch.cuda.set_stream(self.stream)
        self.lib.br_set_streams(self.h, C.c_void_p(self.stream.cuda_stream), None)

    def alloc(self, rows, cols, zero=False):
        return CMat.alloc(self.torch, rows, cols, self.dev, zero)

    def _c(self, rc, what):
        _lib.check(rc, what)

    def panel_stream(self, on: bool):
        self._c(self.lib.br_stream_select(self.h, 1 if on else 0), "stream_select")

    def join(self, waiter_panel: bool):
        self._c(self.lib.br_stream_join(self.h, 1 if waiter_panel else 0), "stream_join")

    def qr_panel(self, P, Y, T, W, tau, lq=False):
        fn = self.lib.br_lq_panel if lq else self.lib.br_qr_panel
        d0, d1 = (P.rows, P.cols)
        self._c(fn(self.h, d0, d1, P.ptr, P.ld, Y.ptr, Y.ld, T.ptr, T.ld,
                   W.ptr if W is not None else None, W.ld if W is not None else 0, tau.ptr),
                "lq_panel" if lq else "qr_panel")

    def gemm(self, Cm, A, B, alpha=1.0, beta=0.0, ta=False, tb=False):
        m, n = Cm.rows, Cm.cols
        k = A.rows if ta else A.cols
        if m == 0 or n == 0:
            return
        self._c(self.lib.br_gemm(self.h, int(ta), int(tb), m, n, k, alpha, A.ptr, A.ld, B.ptr, B.ld,
                                 beta, Cm.ptr, Cm.ld), "gemm")

    def symm_acc(self, X, S, W, alpha=1.0, beta=1.0):
        self._c(self.lib.br_symm_lower_ex(self.h, S.rows, W.cols, alpha, S.ptr, S.ld, W.ptr, W.ld,
                                          beta, X.ptr, X.ld), "symm")

    def syr2k_cols(self, blk, j, cc0, X3, Y):
        """A2[cc0:, cc0:cc0+b] += X3 Y^T + Y X3^T (lower part) where `blk` is the
        locally stored block column holding A2 rows cc0..j-1 of those columns."""
        b = blk.cols
        # a j x j 'virtual' A2 whose columns cc0..cc0+b map onto blk; only
        # lower tiles of that column range are ever touched by the kernel
        fake = blk.ptr - 8 * (cc0 + cc0 * blk.ld)
        self._c(self.lib.br_syr2k_lower(self.h, j, b, C.c_void_p(fake), blk.ld, X3.ptr, X3.ld,
                                        Y.ptr, Y.ld, cc0, cc0 + b), "syr2k")

    def zero(self, M):
        M.t[: M.cols, : M.rows].zero_()

    def copy(self, dst, src):
        dst.t[: dst.cols, : dst.rows].copy_(src.t[: src.cols, : src.rows])

    def sync(self):
        self._c(self.lib.br_sync(self.h), "sync")


class TorchComm:
    """Collectives through torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, dist, group=None):
        self.dist = dist
        self.group = group

    def broadcast(self, M: CMat, src: int):
        # contiguous staging when the view is strided
        t = M.t[: M.cols, : M.rows]
        if t.is_contiguous():
            self.dist.broadcast(t, src=src, group=self.group)
        else:
            c = t.contiguous()
            self.dist.broadcast(c, src=src, group=self.group)
            t.copy_(c)

    def all_reduce(self, M: CMat):
        t = M.t[: M.cols, : M.rows]
        if t.is_contiguous():
            self.dist.all_reduce(t, group=self.group)
        else:
            c = t.contiguous()
            self.dist.all_reduce(c, group=self.group)
            t.copy_(c)

    def all_gather(self, out_list, inp):
        self.dist.all_gather(out_list, inp, group=self.group)


def _sevp_iters(n, w, b):
    ks, k = [], 0
    while n - k - w >= 2:
        ks.append(k)
        k += min(b, n - k - w)
    return ks


def reduce_sym_band_dist(Aloc: CMat, lay: Layout, w: int, ops, comm, lookahead: int = 1):
    """Distributed SEVP on the local block columns `Aloc` (n x ncols_local,
    lower triangle authoritative), in place. Returns the iteration count.
    Band entries of owned columns are final afterwards (use gather_band)."""
    n, b, P, me = lay.n, lay.b, lay.world, lay.rank
    if w != b:
        raise ValueError("the distributed path is built for w == b (the sharded configs)")
    ks = _sevp_iters(n, w, b)
    if not ks:
        return 0
    jmax = n - w
    Yb = [ops.alloc(jmax, b), ops.alloc(jmax, b)]
    Wb = [ops.alloc(jmax, b), ops.alloc(jmax, b)]
    Tb = [ops.alloc(b, b, zero=True), ops.alloc(b, b, zero=True)]
    taub = [ops.alloc(b, 1), ops.alloc(b, 1)]
    X1 = ops.alloc(jmax, b)
    X3 = ops.alloc(jmax, b)
    X2 = ops.alloc(b, b)

    def block(t, r0):  # local block column t, rows r0..n
        s = lay.slot(t)
        return Aloc.view(r0, n, s * b, (s + 1) * b)

    prefetched = False
    for idx, k in enumerate(ks):
        t = k // b
        j = n - k - w
        par = idx & 1
        Y, W, T, tau = Yb[par].view(0, j, 0, b), Wb[par].view(0, j, 0, b), Tb[par], taub[par]
        owner = lay.owner(t)
        if me == owner:
            if prefetched:
                ops.join(waiter_panel=False)
            else:
                ops.qr_panel(block(t, k + w), Y, T, None, tau)
        prefetched = False
        comm.broadcast(Y, owner)
        comm.broadcast(T, owner)
        ops.gemm(W, Y, T)  # same kernel on every rank -> identical W everywhere
        # ---- X1 = sym(A2) W, owned block columns only, then all-reduce ----
        Xv = X1.view(0, j, 0, b)
        ops.zero(Xv)
        mine = [c for c in lay.owned if c > t]
        for c in mine:
            cc0 = c * b - (k + w)
            cc1 = cc0 + b
            blk = block(c, c * b)
            ops.symm_acc(Xv.view(cc0, cc1, 0, b), blk.view(0, b, 0, b), W.view(cc0, cc1, 0, b))
            if cc1 < j:
                below = blk.view(b, n - c * b, 0, b)
                ops.gemm(Xv.view(cc1, j, 0, b), below, W.view(cc0, cc1, 0, b), 1.0, 1.0)
                ops.gemm(Xv.view(cc0, cc1, 0, b), below, W.view(cc1, j, 0, b), 1.0, 1.0, ta=True)
        comm.all_reduce(Xv)
        X2v, X3v = X2, X3.view(0, j, 0, b)
        ops.gemm(X2v, Xv, W, 0.5, 0.0, ta=True)
        ops.copy(X3v, Xv)
        ops.gemm(X3v, Y, X2v, 1.0, 1.0)
        # ---- SYR2K on owned columns; look-ahead on the next panel's owner ----
        nxt = ks[idx + 1] // b if idx + 1 < len(ks) else None
        order = list(mine)
        if lookahead and nxt is not None and lay.owner(nxt) == me and nxt in order:
            cc0 = nxt * b - (k + w)
            ops.syr2k_cols(block(nxt, nxt * b), j, cc0, X3v, Y)
            order.remove(nxt)
            kn = ks[idx + 1]
            jn = n - kn - w
            ops.join(waiter_panel=True)
            ops.panel_stream(True)
            ops.qr_panel(block(nxt, kn + w), Yb[par ^ 1].view(0, jn, 0, b), Tb[par ^ 1], None,
                         taub[par ^ 1])
            ops.panel_stream(False)
            prefetched = True
        for c in order:
            cc0 = c * b - (k + w)
            ops.syr2k_cols(block(c, c * b), j, cc0, X3v, Y)
    return len(ks)


def reduce_tri_band_dist(Aloc: CMat, lay: Layout, w: int, ops, comm, lookahead: int = 1):
    """Distributed upper triangular-band reduction of a square n x n matrix
    held as local block columns, in place. Returns the iteration count."""
    n, b, P, me = lay.n, lay.b, lay.world, lay.rank
    m = n
    if w != b:
        raise ValueError("the distributed path is built for w == b (the sharded configs)")
    torch = ops.torch
    Yu = [ops.alloc(m, b), ops.alloc(m, b)]
    Wu = [ops.alloc(m, b), ops.alloc(m, b)]
    Tu = [ops.alloc(b, b, zero=True), ops.alloc(b, b, zero=True)]
    tauu = [ops.alloc(b, 1), ops.alloc(b, 1)]
    Yv, Wv, Tv, tauv = ops.alloc(n, b), ops.alloc(n, b), ops.alloc(b, b, zero=True), ops.alloc(b, 1)
    Zl = ops.alloc(b, max(b, lay.ncols_local))
    Zr = ops.alloc(m, b)
    rowp = ops.alloc(b, n)  # gathered LQ row panel (b x jr)
    Yg = ops.alloc(lay.ncols_local + b, b)  # Y_V / W_V rows of the owned blocks, gathered
    Wg = ops.alloc(lay.ncols_local + b, b)

    def block(t, r0, r1=None):
        s = lay.slot(t)
        return Aloc.view(r0, m if r1 is None else r1, s * b, (s + 1) * b)

    def blocks(s0, r0, r1=None):
        """Owned block columns from local slot s0 on: one contiguous local range."""
        return Aloc.view(r0, m if r1 is None else r1, s0 * b, lay.ncols_local)

    its = []
    k = 0
    while m - k >= 2 and k < n:
        its.append(k)
        k += b
    prefetched = False
    for idx, k in enumerate(its):
        t = k // b
        i = m - k
        par = idx & 1
        Y, W, T, tau = Yu[par].view(0, i, 0, b), Wu[par].view(0, i, 0, b), Tu[par], tauu[par]
        owner = lay.owner(t)
        if me == owner:
            if prefetched:
                ops.join(waiter_panel=False)
            else:
                ops.qr_panel(block(t, k), Y, T, None, tau)
        prefetched = False
        comm.broadcast(Y, owner)
        comm.broadcast(T, owner)
        ops.gemm(W, Y, T)  # same kernel on every rank -> identical W everywhere
        mine = [c for c in lay.owned if c > t]
        nown = len(mine)
        s0 = lay.slot(mine[0]) if nown else lay.ncols_local // b
        # ---- left update of all owned trailing block columns (one local range) ----
        if nown:
            E = blocks(s0, k)
            Z = Zl.view(0, b, 0, nown * b)
            ops.gemm(Z, W, E, 1.0, 0.0, ta=True)
            ops.gemm(E, Y, Z, 1.0, 1.0)
        jr = n - k - w
        if jr < 1:
            continue
        # ---- LQ row panel: all-gather the owned b x b pieces, factor everywhere ----
        nb_right = (n - (k + b)) // b  # blocks t+1 .. nblk-1
        per = -(-nb_right // P)  # max blocks any rank owns among t+1..
        stage = torch.zeros((P, per * b, b), dtype=torch.float64, device=Aloc.t.device)
        if nown:
            stage[me, : nown * b].copy_(Aloc.t[s0 * b: lay.ncols_local, k: k + b])
        parts = [torch.empty_like(stage[0]) for _ in range(P)]
        comm.all_gather(parts, stage[me].contiguous())
        R = rowp.view(0, b, 0, jr)
        R3 = rowp.t[: nb_right * b].view(nb_right, b, rowp.t.shape[1])
        for r in range(P):
            first = (r - (t + 1)) % P  # first block t+1+first owned by rank r
            cnt = len(range(first, nb_right, P))
            if cnt:
                R3[first::P, :, :b].copy_(parts[r][: cnt * b].view(cnt, b, b))
        Yvv, Wvv = Yv.view(0, jr, 0, b), Wv.view(0, jr, 0, b)
        ops.qr_panel(R, Yvv, Tv, Wvv, tauv, lq=True)
        if lay.owner(t + 1) == me:  # L into block t+1's rows k..k+b
            ops.copy(block(t + 1, k, k + b), R.view(0, b, 0, b))
        # ---- right update: partial Z over owned columns, all-reduce, local apply ----
        Zv = Zr.view(0, i - b, 0, b)
        if nown:
            # rows of Y_V / W_V belonging to the owned blocks, in local order
            first = (me - (t + 1)) % P
            Yg3 = Yg.t[:b, : nown * b].view(b, nown, b)
            Wg3 = Wg.t[:b, : nown * b].view(b, nown, b)
            Yv3 = Yv.t[:b, : nb_right * b].view(b, nb_right, b)
            Wv3 = Wv.t[:b, : nb_right * b].view(b, nb_right, b)
            Yg3.copy_(Yv3[:, first::P, :])
            Wg3.copy_(Wv3[:, first::P, :])
            ops.gemm(Zv, blocks(s0, k + b), Wg.view(0, nown * b, 0, b), 1.0, 0.0)
        else:
            ops.zero(Zv)
        comm.all_reduce(Zv)
        nxt = t + 1 if idx + 1 < len(its) else None
        lead = 0
        if lookahead and nxt is not None and lay.owner(nxt) == me and nown and mine[0] == nxt:
            ops.gemm(block(nxt, k + b), Zv, Yg.view(0, b, 0, b), 1.0, 1.0, tb=True)
            lead = 1
            kn = its[idx + 1]
            ops.join(waiter_panel=True)
            ops.panel_stream(True)
            ops.qr_panel(block(nxt, kn), Yu[par ^ 1].view(0, m - kn, 0, b), Tu[par ^ 1], None,
                         tauu[par ^ 1])
            ops.panel_stream(False)
            prefetched = True
        if nown > lead:
            ops.gemm(blocks(s0 + lead, k + b), Zv, Yg.view(lead * b, nown * b, 0, b), 1.0, 1.0,
                     tb=True)
    return len(its)


def scatter_columns(A: np.ndarray, lay: Layout, ops) -> CMat:
    """Upload this rank's block columns of a host matrix (F-order)."""
    torch = ops.torch
    L = ops.alloc(A.shape[0], lay.ncols_local)
    for q, t in enumerate(lay.owned):
        blk = np.ascontiguousarray(A[:, t * lay.b : (t + 1) * lay.b].T)  # (b, n) row-major
        L.t[q * lay.b : (q + 1) * lay.b, : A.shape[0]].copy_(torch.from_numpy(blk))
    return L


def gather_band(Aloc: CMat, lay: Layout, w: int, kind: str, comm, torch) -> np.ndarray | None:
    """Assemble the band on rank 0: SEVP -> full symmetric band (mirrored,
    off-band exactly 0, ref sevp.py:276-284); triband -> upper band with
    lower bw 0 (ref svd.py:237-239). Other ranks return None."""
    n, b, P = lay.n, lay.b, lay.world
    local = Aloc.t[: lay.ncols_local, :n].contiguous()
    per = -(-lay.nblk // P) * b
    stage = torch.zeros((per, n), dtype=torch.float64, device=Aloc.t.device)
    stage[: lay.ncols_local].copy_(local)
    parts = [torch.empty_like(stage) for _ in range(P)]
    comm.all_gather(parts, stage)
    if lay.rank != 0:
        return None
    full = np.zeros((n, n), order="F")
    for r in range(P):
        host = parts[r].cpu().numpy()
        blks = [t for t in range(lay.nblk) if t % P == r]
        for q, t in enumerate(blks):
            full[:, t * b : (t + 1) * b] = host[q * b : (q + 1) * b, :].T
    ii = np.arange(n)[:, None]
    jj = np.arange(n)[None, :]
    if kind == "sevp":
        low = np.tril(full)
        low[(ii - jj) > w] = 0.0
        out = low + low.T
        out[ii == jj] = np.diag(low)
        return np.asfortranarray(out)
    full[(ii > jj) | (jj > ii + w)] = 0.0
    return full
