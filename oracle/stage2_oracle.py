"""Second stage (band -> tridiagonal / bidiagonal) by bulge chasing: the
sequential NumPy restatement the CUDA kernels are checked against (TEST
ORACLE ONLY; nothing in the product package imports it).

The reference package stops at the band (its spec leaves the second stage
out; the paper motivates it), so
there is no reference output to pin this against: PARITY UNPINNED by the
reference. What pins it instead: LAPACK's eigenvalues / singular values of
the input (orthogonal similarity / equivalence preserves them), exact zeros
outside the tridiagonal / bidiagonal, and the GPU kernels reproducing this
task sequence to rounding.

Algorithm (Householder bulge chasing, one column per sweep; the task
structure of Haidar, Ltaief and Dongarra's two-stage tridiagonal reduction):
every reflector uses the reference's convention (house_gen, ref
kernels.py:86-110: beta = -sign(x0)||x||, tau = 2 on a zero tail), and a
vector of length 1 is left alone.

SEVP, symmetric band of bandwidth w (lower triangle read):
  sweep s, task 0: H = house(S[s+1 : s+1+L, s]) annihilates column s below
      the subdiagonal; D = S[s+1 : s+1+L]^2 := H D H.
  task j >= 1 (block row r = previous block's end, L2 rows):
      O = S[r : r+L2, previous block] := O H   (the bulge appears in O),
      H2 = house(O[:, 0]) annihilates O's first column: O := H2 O,
      D2 = S[r : r+L2]^2 := H2 D2 H2; then H := H2.
SVD, upper triangular band of bandwidth w (m >= n, the top n x n square):
  sweep s, task 0: right reflector on row s (columns s+1 .. s+L), applied
      to rows s .. s+L; left reflector on column s+1 (rows s+1 .. s+L),
      applied to columns s+1 .. s+L+w.
  task j >= 1 (rows r .. r+L of the previous left reflector, fill to the
      right from column c0 = r + L): right reflector on row r's entries
      c0 .. c0+L2 (keeps the band entry at c0), applied to rows r .. c0+L2;
      left reflector on column c0 (rows c0 .. c0+L2), applied to columns
      c0 .. c0+L2+w.
"""
from __future__ import annotations

import numpy as np

from .bandred_oracle import house_gen


def _two_sided(D, v, tau):
    """D := (I - tau v v^T) D (I - tau v v^T) for symmetric D (in place)."""
    y = tau * (D @ v)
    a = 0.5 * tau * float(v @ y)
    wv = y - a * v
    D -= np.outer(v, wv) + np.outer(wv, v)


def sb2st(B, w):
    """Symmetric band (bandwidth w, lower triangle read) -> (d, e, S) with
    S the final tridiagonal working matrix."""
    n = B.shape[0]
    L0 = np.tril(np.asarray(B, dtype=np.float64))
    S = L0 + np.tril(L0, -1).T
    for s in range(n - 2):
        r = s + 1
        L = min(w, n - r)
        if L < 2:
            continue
        v, tau, beta = house_gen(S[r:r + L, s])
        S[r:r + L, s] = 0.0
        S[r, s] = beta
        S[s, r:r + L] = S[r:r + L, s]
        _two_sided(S[r:r + L, r:r + L], v, tau)
        while True:
            rb = r + L
            L2 = min(w, n - rb)
            if L2 <= 0:
                break
            O = S[rb:rb + L2, r:r + L]
            O -= np.outer(O @ v, tau * v)
            if L2 >= 2:
                v2, tau2, beta2 = house_gen(O[:, 0])
                O[:, 0] = 0.0
                O[0, 0] = beta2
                O[:, 1:] -= np.outer(v2, tau2 * (v2 @ O[:, 1:]))
            S[r:r + L, rb:rb + L2] = O.T
            if L2 < 2:
                break
            _two_sided(S[rb:rb + L2, rb:rb + L2], v2, tau2)
            r, L, v, tau = rb, L2, v2, tau2
    return np.diag(S).copy(), np.diag(S, -1).copy(), S


def tb2bd(B, w):
    """Upper triangular band (bandwidth w; m >= n, rows >= n zero) ->
    (d, e, Bw) with Bw the final upper bidiagonal n x n working matrix."""
    m, n = B.shape
    if m < n:
        raise ValueError("tb2bd: m >= n (reduce the transpose)")
    A = np.triu(np.asarray(B, dtype=np.float64)[:n, :n]).copy()
    for s in range(n - 1):
        # task 0: row s
        L = min(w, n - s - 1)
        if L >= 2:
            v, tau, beta = house_gen(A[s, s + 1:s + 1 + L])
            A[s, s + 1:s + 1 + L] = 0.0
            A[s, s + 1] = beta
            R = A[s + 1:s + 1 + L, s + 1:s + 1 + L]
            R -= np.outer(R @ v, tau * v)
        if L < 1:
            continue
        # left reflector on column s + 1, rows s+1 .. s+L
        r = s + 1
        Lr = min(w, n - r)
        if Lr < 2:
            continue
        u, tu, bu = house_gen(A[r:r + Lr, r])
        A[r:r + Lr, r] = 0.0
        A[r, r] = bu
        c1 = min(n, r + Lr + w)
        M = A[r:r + Lr, r + 1:c1]
        M -= np.outer(u, tu * (u @ M))
        # chase
        while True:
            c0 = r + Lr
            L2 = min(w, n - c0)
            if L2 <= 0:
                break
            # right reflector on row r, columns c0 .. c0+L2
            if L2 >= 2:
                v, tau, beta = house_gen(A[r, c0:c0 + L2])
                A[r, c0:c0 + L2] = 0.0
                A[r, c0] = beta
                rows = A[r + 1:c0 + L2, c0:c0 + L2]
                rows -= np.outer(rows @ v, tau * v)
            # left reflector on column c0, rows c0 .. c0+L2
            if L2 < 2:
                break
            u, tu, bu = house_gen(A[c0:c0 + L2, c0])
            A[c0:c0 + L2, c0] = 0.0
            A[c0, c0] = bu
            c1 = min(n, c0 + L2 + w)
            M = A[c0:c0 + L2, c0 + 1:c1]
            M -= np.outer(u, tu * (u @ M))
            r, Lr = c0, L2
    return np.diag(A).copy(), np.diag(A, 1).copy(), A
