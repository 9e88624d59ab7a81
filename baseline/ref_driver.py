"""Times the REFERENCE implementation itself on the host cores (bench only).

The reference package (`bandred`, pure Python + NumPy) is installed once,
offline, into baseline/_ref by the base contract's recipe

    python -m pip install --no-index --no-build-isolation --no-deps \
        --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>

(baseline/_ref is git-ignored and travels to the GPU box with the snapshot).
`bench.py --impl reference` and the `cpu_baseline` leg call the reference's
own public entry points (`reduce_tri_band`, `reduce_sym_band`, ref
svd.py:205, sevp.py:287) on the bench's input, bounded to the first K panels
so that a step stays within seconds:
  * triangular band: the reference's sequential loop (ref svd.py:179-202) is
    stopped after K panel tasks (QR and LQ panels each count, with the
    one-sided update that follows each) by counting wrappers around its
    `qr_panel` / `lq_panel`;
  * SEVP: its schedule (ref sevp.py:110-118) is truncated to K iterations.
Two arithmetic modes:
  * "pure": the reference unmodified (its `matmul` is a sequential rank-1
    loop, ref kernels.py:39-83, ~0.2 GFLOP/s);
  * "blas": the reference code with only `matmul` rebound to multithreaded
    BLAS (SURVEY.md 8(c) tier B: agrees with the pure reference to ~5e-14),
    the fastest the reference's algorithm runs on these cores.
Rates use the reference's own FLOPS counter (ref flops.py) over the sampled
iterations.
"""
from __future__ import annotations

import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


class _Stop(Exception):
    pass


def available() -> bool:
    return os.path.isdir(os.path.join(REF, "bandred"))


def load(mode: str = "blas"):
    """Import the installed reference; mode "blas" rebinds its matmul."""
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import numpy as np

    import bandred
    import bandred.kernels as K
    import bandred.sevp as S
    import bandred.svd as V

    if not hasattr(K, "_pure_matmul"):
        K._pure_matmul = K.matmul
    if mode == "blas":
        FL = K.FLOPS

        def blas_matmul(alpha, A, B, beta, C, workers=None):
            m, k = A.shape
            n = B.shape[1]
            if beta == 0.0:
                C[...] = 0.0
            elif beta != 1.0:
                np.multiply(C, beta, out=C)
            if alpha == 0.0 or k == 0 or m == 0 or n == 0:
                return C
            FL.add("matmul", 2 * m * k * n)
            P = A @ B
            if alpha != 1.0:
                P *= alpha
            C += P
            return C

        fn = blas_matmul
    else:
        fn = K._pure_matmul
    for mod in (K, S, V):
        mod.matmul = fn
    return bandred


def sample(bandred, kind, A, n, w, b, iters, workers=None):
    """Run the reference on A for its first `iters` panel tasks (SEVP:
    iterations; triangular band: QR / LQ panels with their updates); returns
    (counted flops, seconds, panel tasks done)."""
    groups = bandred.ExecGroups(workers, 1) if workers and workers > 1 else None
    before = bandred.FLOPS.snapshot()
    t0 = time.perf_counter()
    done = 0
    try:
        if kind == "sevp":
            import bandred.sevp as S

            orig_sched, orig_fin = S._schedule, S._finalize
            S._schedule = lambda nn, ww, bb: orig_sched(nn, ww, bb)[:iters]
            S._finalize = lambda AA, nn, ww: AA  # the sample stops mid-reduction
            try:
                cfg = bandred.SevpConfig(n, w, b, bandred.SevpVariant.REFERENCE)
                r = bandred.reduce_sym_band(A, cfg, groups)
                done = r.iterations
            finally:
                S._schedule, S._finalize = orig_sched, orig_fin
        else:
            import bandred.svd as V

            oq, ol = V.qr_panel, V.lq_panel
            count = [0]

            def counted(fn):
                def f(P, inner_b=16):
                    if count[0] >= iters:
                        raise _Stop()
                    count[0] += 1
                    return fn(P, inner_b)

                return f

            V.qr_panel, V.lq_panel = counted(oq), counted(ol)
            try:
                bandred.reduce_tri_band(A, w, b, groups)
            except _Stop:
                pass
            finally:
                V.qr_panel, V.lq_panel = oq, ol
            done = count[0]
    finally:
        if groups is not None:
            groups.close()
    dt = time.perf_counter() - t0
    after = bandred.FLOPS.snapshot()
    flops = sum(after.get(k, 0) - before.get(k, 0) for k in after if k != "total")
    return flops, dt, done
