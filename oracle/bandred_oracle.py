"""NumPy restatement of the reference `bandred` hot path (TEST ORACLE ONLY).

Every function cites the reference file:line it restates (paths relative to
the reference package `pkg/src/bandred/`). Arithmetic differences from the
reference are deliberate and limited to summation order: the reference's
`matmul` (kernels.py:39-83) is a sequential rank-1 loop without FMA, this
oracle uses BLAS `@`. The survey measured that swap at 4.5e-14 (SEVP) and
5.6e-14 (triband) relative Frobenius at n=2048, far inside the 1e-12*sqrt(n)
parity bound. Sign conventions (house_gen zero-tail rule, T = -T_larft) are
restated exactly, because parity depends on them.

Nothing in the product package imports this module.
"""
from __future__ import annotations

import numpy as np

_BLK = 1024  # column block of the blocked SYMM / SYR2K restatements

__all__ = [
    "house_gen",
    "qr_panel",
    "lq_panel",
    "build_w",
    "t_from_gram",
    "apply_wy_left",
    "apply_wy_right",
    "symm_lower",
    "syr2k_lower",
    "sym_two_sided_update",
    "sevp_schedule",
    "tri_schedule",
    "reduce_sym_band",
    "reduce_tri_band",
    "reduce_band_svd",
    "band_schedule",
    "finalize_sym",
    "mask_tri_band",
    "band_check",
    "sevp_nominal_flops",
    "svd_nominal_flops",
    "gen_c1",
    "gen_c2",
    "gen_c3",
    "gen_c4",
    "gen_c5",
    "gen_config",
]


# --------------------------------------------------------------------------
# kernels (reference kernels.py)
# --------------------------------------------------------------------------


def house_gen(x):
    """Reflector (v, tau, beta) with (I - tau v v^T) x = beta e1.

    Restates kernels.py:86-110: beta = -sign(x0)*||x|| with x0 == 0 treated
    as positive, applied even when the tail is zero (tau = 2); the zero
    vector gives tau = beta = 0 and v = e1. ||x|| is sqrt(x.x) as in
    np.linalg.norm (kernels.py:101).
    """
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 1 or x.size < 1:
        raise ValueError("house_gen needs a vector of length >= 1")
    v = np.zeros(x.size)
    v[0] = 1.0
    nrm = float(np.sqrt(np.dot(x, x)))
    if nrm == 0.0:
        return v, 0.0, 0.0
    sign = -1.0 if x[0] < 0 else 1.0
    beta = -sign * nrm
    v0 = x[0] - beta
    v[1:] = x[1:] / v0
    tau = (beta - x[0]) / beta
    return v, float(tau), float(beta)


def build_w(Y, T):
    """W = Y T (kernels.py:139-149)."""
    return np.asfortranarray(Y @ T)


def t_from_gram(G, tau):
    """Compact-WY T from the Gram matrix G = Y^T Y and tau.

    Restates _t_extend (kernels.py:152-162) column by column:
    T[0:i, i] = -tau_i * T[0:i, 0:i] @ G[0:i, i], T[i, i] = -tau_i
    (i.e. T = -T_larft).
    """
    b = len(tau)
    T = np.zeros((b, b), order="F")
    for i in range(b):
        if i > 0:
            T[:i, i] = -tau[i] * (T[:i, :i] @ G[:i, i])
        T[i, i] = -tau[i]
    return T


def qr_panel(P, inner_b=16):
    """Blocked left-looking Householder QR of a j x b panel, in place.

    Restates kernels.py:165-208. Returns (Y, T, W, R, tau); P's top b x b
    holds R and the reflector tails sit below it, as in the reference.
    """
    j, b = P.shape
    if j < b or b < 1:
        raise ValueError(f"qr_panel needs j >= b >= 1, got {j} x {b}")
    if inner_b < 1:
        raise ValueError("inner_b >= 1")
    Y = np.zeros((j, b), order="F")
    T = np.zeros((b, b), order="F")
    tau = np.zeros(b)
    for s in range(0, b, inner_b):
        e = min(s + inner_b, b)
        if s > 0:  # kernels.py:183-191 (left-looking block application)
            blk = P[:, s:e]
            blk += Y[:, :s] @ (T[:s, :s].T @ (Y[:, :s].T @ blk))
        for i in range(s, e):  # kernels.py:192-205
            v, ti, beta = house_gen(P[i:, i].copy())
            tau[i] = ti
            Y[i:, i] = v
            P[i, i] = beta
            P[i + 1 :, i] = v[1:]
            if i + 1 < e and ti != 0.0:
                rest = P[i:, i + 1 : e]
                rest -= ti * np.outer(v, v @ rest)
            if i > 0:  # _t_extend, kernels.py:152-162
                T[:i, i] = -ti * (T[:i, :i] @ (Y[i:, :i].T @ Y[i:, i]))
            T[i, i] = -ti
    W = build_w(Y, T)
    R = np.triu(P[:b, :b]).copy(order="F")
    return Y, T, W, R, tau


def lq_panel(P, inner_b=16):
    """Blocked left-looking LQ of a b x j panel, in place (kernels.py:211-255).

    Reflectors act on rows; V = I + W Y^T is applied from the right.
    Returns (Y, T, W, L, tau) with Y of shape j x b.
    """
    b, j = P.shape
    if j < b or b < 1:
        raise ValueError(f"lq_panel needs b x j with j >= b >= 1, got {b} x {j}")
    if inner_b < 1:
        raise ValueError("inner_b >= 1")
    Y = np.zeros((j, b), order="F")
    T = np.zeros((b, b), order="F")
    tau = np.zeros(b)
    for s in range(0, b, inner_b):
        e = min(s + inner_b, b)
        if s > 0:  # kernels.py:231-239
            blk = P[s:e, :]
            blk += ((blk @ Y[:, :s]) @ T[:s, :s]) @ Y[:, :s].T
        for i in range(s, e):  # kernels.py:240-252
            v, ti, beta = house_gen(P[i, i:].copy())
            tau[i] = ti
            Y[i:, i] = v
            P[i, i] = beta
            P[i, i + 1 :] = v[1:]
            if i + 1 < e and ti != 0.0:
                rest = P[i + 1 : e, i:]
                rest -= ti * np.outer(rest @ v, v)
            if i > 0:
                T[:i, i] = -ti * (T[:i, :i] @ (Y[i:, :i].T @ Y[i:, i]))
            T[i, i] = -ti
    W = build_w(Y, T)
    L = np.tril(P[:b, :b]).copy(order="F")
    return Y, T, W, L, tau


def apply_wy_left(A, Y, W):
    """A := A + Y (W^T A), in place (kernels.py:258-284)."""
    if A.shape[0] == 0 or A.shape[1] == 0:
        return A
    Z = W.T @ A
    A += (Z.T @ Y.T).T  # the product formed F-ordered, like A (a C-ordered
    return A             # temporary makes the in-place add stride-bound)


def apply_wy_right(A, Y, W):
    """A := A + (A W) Y^T, in place (kernels.py:287-309)."""
    if A.shape[0] == 0 or A.shape[1] == 0:
        return A
    AW = A @ W
    A += (Y @ AW.T).T
    return A


def symm_lower(A2, W):
    """sym(A2) W reading only A2's lower triangle (kernels.py:312-341)."""
    j = A2.shape[0]
    X1 = np.zeros((j, W.shape[1]), order="F")
    for a in range(0, j, _BLK):  # column blocks: only lower-stored entries are read
        e = min(j, a + _BLK)
        D = np.tril(A2[a:e, a:e])
        X1[a:e] += D @ W[a:e] + np.tril(D, -1).T @ W[a:e]
        if e < j:
            S = A2[e:, a:e]  # strictly below the diagonal block
            X1[e:] += S @ W[a:e]
            X1[a:e] += S.T @ W[e:]
    return X1


def syr2k_lower(A2, X3, Y, c0, c1):
    """A2[:, c0:c1] += X3 Y^T + Y X3^T on the lower triangle only, in place
    (kernels.py:344-378). Entries above the diagonal are left untouched."""
    j = A2.shape[0]
    if not (0 <= c0 <= c1 <= j):
        raise ValueError("syr2k_lower bad column range")
    if c0 == c1:
        return A2
    for a in range(c0, c1, _BLK):  # column blocks; lower part of each only
        e = min(c1, a + _BLK)
        # rows a.. x cols a..e, formed F-ordered: (Y_b X3^T + X3_b Y^T)^T
        upd = (Y[a:e] @ X3[a:].T + X3[a:e] @ Y[a:].T).T
        d = np.tril(np.ones((e - a, e - a), dtype=bool))
        A2[a:e, a:e][d] += upd[: e - a][d]
        A2[e:, a:e] += upd[e - a :]
    return A2


def sym_two_sided_update(A2, Y, W):
    """A2 := Q^T A2 Q on the lower triangle, Q = I + W Y^T (kernels.py:381-401).

    X1 = sym(A2) W; X2 = (1/2) X1^T W; X3 = X1 + Y X2; A2 += X3 Y^T + Y X3^T.
    Returns X3 as well (useful for kernel-level parity).
    """
    j = A2.shape[0]
    if j == 0 or Y.shape[1] == 0:
        return A2, None
    X1 = symm_lower(A2, W)
    X2 = 0.5 * (X1.T @ W)
    X3 = X1 + Y @ X2
    syr2k_lower(A2, X3, Y, 0, j)
    return A2, X3


# --------------------------------------------------------------------------
# reductions (reference sevp.py / svd.py)
# --------------------------------------------------------------------------


def sevp_schedule(n, w, b):
    """Leading columns of all SEVP iterations (sevp.py:110-118)."""
    ks, k = [], 0
    while n - k - w >= 2:
        ks.append(k)
        k += min(b, n - k - w)
    return ks


def tri_schedule(m, n, b):
    """(k, bp) of all triangular-band iterations, m >= n (svd.py:179-202)."""
    out, k = [], 0
    while m - k >= 2 and k < n:
        bp = min(b, n - k, m - k)
        out.append((k, bp))
        k += bp
    return out


def finalize_sym(A, n, w):
    """Mirror lower -> upper and zero off-band exactly (sevp.py:276-284)."""
    out = np.zeros((n, n), order="F")
    for c in range(n):  # lower in-band entries kept, upper ones mirrored
        lo = A[c : min(n, c + w + 1), c]
        out[c : c + lo.size, c] = lo
        out[c, c + 1 : c + lo.size] = lo[1:]
    return out


def mask_tri_band(A, w):
    """Zero i > j and j > i + w exactly (svd.py:237-239)."""
    m, n = A.shape
    for c in range(n):  # column by column (no m x n index masks)
        A[c + 1 :, c] = 0.0
        if c - w > 0:
            A[: c - w, c] = 0.0
    return A


def reduce_sym_band(A, n, w, b, inner_b=16, accumulate_q=False, max_iters=None, finalize=True,
                    factors=None):
    """Dense symmetric -> symmetric band, Reference schedule.

    Restates reduce_sym_band (sevp.py:287-324) with _run_reference
    (sevp.py:194-206) and the task bodies sevp.py:128-188. Reads only the
    lower triangle. Returns (band, q, iterations); n <= w+1 returns the
    copied input unchanged (sevp.py:302-305). Test hooks: `max_iters` stops
    after that many panels, `finalize=False` returns the raw working matrix
    (the partial-reduction comparison of BR_OPT_MAX_ITERS), `factors` (a
    dict) receives k -> (Y, T, tau) of every panel (state.factors[k],
    sevp.py:128-134).
    """
    if not (1 <= b <= w) or n < 1:
        raise ValueError("need n >= 1, 1 <= b <= w")
    A = np.array(A, dtype=np.float64, order="F")
    if A.shape != (n, n):
        raise ValueError("shape mismatch")
    ks = sevp_schedule(n, w, b)
    if not ks:
        return A, None, 0
    Q = np.eye(n, order="F") if accumulate_q else None
    if max_iters is not None:  # bounded CPU-baseline sample (bench.py)
        ks = ks[:max_iters]
    for k in ks:
        bp = min(b, n - k - w)
        j = n - k - w
        Y, T, W, R, tau = qr_panel(A[k + w : n, k : k + bp], inner_b)
        if factors is not None:
            factors[k] = (Y, T, tau)
        if Q is not None:
            apply_wy_right(Q[:, k + w : n], Y, W)
        if bp < w:
            apply_wy_left(A[k + w : n, k + bp : k + w], Y, W)
        A2 = A[k + w : n, k + w : n]
        X1 = symm_lower(A2, W)
        X2 = 0.5 * (X1.T @ W)
        X3 = X1 + Y @ X2
        syr2k_lower(A2, X3, Y, 0, j)
    if not finalize:
        return A, Q, len(ks)
    return finalize_sym(A, n, w), Q, len(ks)


def reduce_tri_band(A, w, b, inner_b=16, max_iters=None, finalize=True, factors=None):
    """Dense general -> upper triangular-band (svd.py:179-247).

    Returns (band, lower_bw, upper_bw, iterations); m < n reduces A^T and
    transposes back (svd.py:221-232). Test hooks as in reduce_sym_band;
    `factors` receives ("qr", k) / ("lq", k) -> (Y, T, tau) (fu / fv,
    svd.py:185,195).
    """
    if w < 1 or not (1 <= b <= w):
        raise ValueError("need w >= 1, 1 <= b <= w")
    A = np.array(A, dtype=np.float64, order="F")
    if A.ndim != 2:
        raise ValueError("reduce_tri_band needs a 2-D matrix")
    m, n = A.shape
    if m < n:
        band, _, _, it = reduce_tri_band(np.asfortranarray(A.T), w, b, inner_b)
        return np.asfortranarray(band.T), w, 0, it
    it = 0
    sched = tri_schedule(m, n, b)
    if max_iters is not None:  # bounded CPU-baseline sample (bench.py)
        sched = sched[:max_iters]
    for k, bp in sched:
        Yu, Tu, Wu, _, tu = qr_panel(A[k:m, k : k + bp], inner_b)
        if factors is not None:
            factors[("qr", k)] = (Yu, Tu, tu)
        apply_wy_left(A[k:m, k + bp : n], Yu, Wu)
        jr = n - k - w
        if jr >= 1:
            bq = min(bp, jr)
            Yv, Tv, Wv, _, tv = lq_panel(A[k : k + bq, k + w : n], inner_b)
            if factors is not None:
                factors[("lq", k)] = (Yv, Tv, tv)
            apply_wy_right(A[k + bq : m, k + w : n], Yv, Wv)
        it += 1
    if not finalize:
        return A, 0, w, it
    return mask_tri_band(A, w), 0, w, it


def band_schedule(m, n, w, b):
    """(k, bp, jr, bq) of the equal-bandwidth band form (svd.py:265-278)."""
    out, k = [], 0
    while m - k - w >= 2 and k < n:
        bp = min(b, m - k - w, n - k)
        jr = n - k - w
        bq = min(bp, jr) if jr >= 1 else 0
        out.append((k, bp, jr, bq))
        k += bp
    return out


def reduce_band_svd(A, w, b, simultaneous=False, inner_b=16):
    """Dense general -> band with lower = upper bandwidth w (svd.py:515-589).

    Reference order (svd.py:359-373): QR(B0), left(B1), left(D), LQ(C0),
    right(C1), right(D). Simultaneous (svd.py:376-391, 317-356): the two D
    applications fused, Z_L = D^T W_U, Z_R = D W_V, X = Z_R + Y_U (Z_L^T W_V),
    D += X Y_V^T + Y_U Z_L^T. m < n reduces A^T; m <= w + 1 returns the copy
    unchanged. Returns (band, lower_bw, upper_bw, iterations).
    """
    A = np.array(A, dtype=np.float64, order="F")
    m, n = A.shape
    if m < n:
        band, lo, up, it = reduce_band_svd(np.asfortranarray(A.T), w, b, simultaneous, inner_b)
        return np.asfortranarray(band.T), up, lo, it
    sched = band_schedule(m, n, w, b)
    if not sched:
        return A, w, w, 0
    for k, bp, jr, bq in sched:
        Yu, Tu, Wu, _, _ = qr_panel(A[k + w : m, k : k + bp], inner_b)
        b1end = min(k + w, n)
        if k + bp < b1end:
            apply_wy_left(A[k + w : m, k + bp : b1end], Yu, Wu)
        if jr < 1:
            continue
        D = A[k + w : m, k + w : n]
        if not simultaneous:
            apply_wy_left(D, Yu, Wu)
        Yv, Tv, Wv, _, _ = lq_panel(A[k : k + bq, k + w : n], inner_b)
        if k + bq < k + w:
            apply_wy_right(A[k + bq : k + w, k + w : n], Yv, Wv)
        if not simultaneous:
            apply_wy_right(D, Yv, Wv)
        else:
            ZL = D.T @ Wu
            ZR = D @ Wv
            X = ZR + Yu @ (ZL.T @ Wv)
            D += X @ Yv.T
            D += Yu @ ZL.T
    i = np.arange(m)[:, None]
    jj = np.arange(n)[None, :]
    A[np.abs(i - jj) > w] = 0.0
    return A, w, w, len(sched)


def band_check(B, lower_bw, upper_bw):
    """Exact max |entry| outside the band (oracles.py:123-135)."""
    B = np.asarray(B)
    m, n = B.shape
    i = np.arange(m)[:, None]
    j = np.arange(n)[None, :]
    mask = (i - j > lower_bw) | (j - i > upper_bw)
    if not mask.any():
        return 0.0
    return float(np.max(np.abs(B[mask])))


def sevp_nominal_flops(n):
    """4 n^3 / 3 (sevp.py:92-96)."""
    if n < 0:
        raise ValueError("n >= 0")
    return round(4 * n**3 / 3)


def svd_nominal_flops(m, n):
    """4 (m n^2 - n^3 / 3), m >= n (svd.py:127-132)."""
    if n < 0 or m < n:
        raise ValueError("need m >= n >= 0")
    return round(4 * (m * n * n - n**3 / 3))


# --------------------------------------------------------------------------
# BASELINE.json inputs, seeded synthetic, F-order
# --------------------------------------------------------------------------


def gen_c1(n=2048):
    g = np.random.default_rng(0).standard_normal((n, n))
    return np.asfortranarray((g + g.T) / 2.0)


def gen_c2(n=2048):
    return np.asfortranarray(np.random.default_rng(1).standard_normal((n, n)))


def gen_c3(n=8192):
    q, _ = np.linalg.qr(np.random.default_rng(2).standard_normal((n, n)))
    s = np.random.default_rng(3).choice([-1.0, 1.0], n)
    lam = 10.0 ** (-8.0 * np.arange(n) / (n - 1)) * s
    a = (q * lam) @ q.T
    return np.asfortranarray((a + a.T) / 2.0)


def gen_c4(n=16384):
    return np.asfortranarray(np.random.default_rng(4).uniform(-1.0, 1.0, (n, n)))


def gen_c5(n=32768):
    g = np.random.default_rng(5).standard_normal((n, n))
    g += g.T
    g *= 0.5
    return np.asfortranarray(g)


def gen_config(name, n=None):
    f = {"c1": gen_c1, "c2": gen_c2, "c3": gen_c3, "c4": gen_c4, "c5": gen_c5}[name]
    return f() if n is None else f(n)
