"""Dense symmetric -> symmetric band on the B200 (drop-in for ref sevp.py).

`reduce_sym_band(A, cfg, groups=None)` keeps the reference's signature,
validation, result type and edge semantics (ref sevp.py:287-324):
  * only A's lower triangle is read; A itself is never mutated;
  * the band is returned in full storage, mirrored, off-band exactly 0;
  * n <= w + 1 returns the copied input unchanged (not symmetrized),
    q=None, flops {"total": 0}, iterations 0.
Schedules: REFERENCE -> look-ahead depth 0; V1 / V2 -> depth 1 (the next
panel is factored on the panel stream while the trailing update finishes).
Both are bitwise identical on the GPU. Extensions (keyword-only):
`lookahead` overrides the depth, `device` selects the GPU, `return_factors`
returns every panel's Householder factors (`result.factors`, see factors.py;
the reference keeps them only in private state, ref sevp.py:106,128-134).
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _dev, _lib
from . import factors as _factors
from . import multi as _multi
from .flops import FLOPS, apply_correction, sevp_counted_flops, sevp_nominal_flops, tau_zero_correction  # noqa: F401


class SevpVariant(Enum):
    REFERENCE = "reference"
    V1 = "v1"
    V2 = "v2"


class V2Mapping(Enum):
    ON_TS = "on_ts"
    ON_ALL = "on_all"


@dataclass
class SevpConfig:
    n: int
    w: int
    b: int
    variant: SevpVariant = SevpVariant.REFERENCE
    v2_mapping: V2Mapping = V2Mapping.ON_TS
    accumulate_q: bool = False
    inner_b: int = 16

    def validate(self):
        """Same rules and messages as ref sevp.py:66-81."""
        if self.n < 1:
            raise ValueError("n >= 1")
        if self.w < 1:
            raise ValueError("w >= 1")
        if not (1 <= self.b <= self.w):
            raise ValueError("need 1 <= b <= w")
        if self.variant == SevpVariant.V1 and 2 * self.b > self.w:
            raise ValueError(f"V1 requires 2b <= w, got b={self.b}, w={self.w}")
        if self.variant == SevpVariant.V2 and 2 * self.b <= self.w:
            warnings.warn(
                f"V2 with 2b <= w (b={self.b}, w={self.w}) is valid but outside "
                "its intended regime; V1 covers this case",
                RuntimeWarning,
                stacklevel=3,
            )


@dataclass
class SevpResult:
    band: np.ndarray
    q: np.ndarray | None
    flops: dict
    iterations: int
    factors: "_factors.BandFactors | None" = None  # extension: return_factors=True


def _schedule(n, w, b):
    """Leading columns of all iterations (ref sevp.py:110-118)."""
    ks = []
    k = 0
    while n - k - w >= 2:
        ks.append(k)
        k += min(b, n - k - w)
    return ks


def _depth(cfg, groups, lookahead):
    if lookahead is not None:
        if lookahead not in (0, 1):
            raise ValueError("lookahead must be 0 or 1 (depth > 1 is a reference non-goal)")
        return int(lookahead)
    if groups is not None and getattr(groups, "ts_count", 1) == 0:
        return 0
    return 0 if cfg.variant == SevpVariant.REFERENCE else 1


def reduce_sym_band(A, cfg, groups=None, *, lookahead=None, device=None, stats=None,
                    return_factors=False, ngpus=None, devices=None):
    """Reduce symmetric A to a symmetric band matrix of bandwidth cfg.w.

    ngpus / devices (extension): run the 1D block-cyclic
    multi-GPU driver over those devices from this one process (multi.py);
    needs w == b and n a multiple of b, without accumulate_q / factors."""
    cfg.validate()
    A = np.array(A, dtype=np.float64, order="F")
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise ValueError("reduce_sym_band needs a square matrix")
    if A.shape[0] != cfg.n:
        raise ValueError(f"cfg.n={cfg.n} does not match matrix order {A.shape[0]}")
    depth = _depth(cfg, groups, lookahead)
    ks = _schedule(cfg.n, cfg.w, cfg.b)
    if not ks:  # n <= w + 1: the copy, unchanged (ref sevp.py:302-305); no arithmetic
        return SevpResult(band=A, q=None, flops={"total": 0}, iterations=0)
    devs = _multi.resolve_devices(ngpus, devices)
    if devs is not None:
        return _reduce_multi(A, cfg, depth, devs, return_factors, stats)
    lib = _lib.load()
    h, _ = _dev.ctx(device)
    n = cfg.n
    band = np.empty((n, n), order="F")
    Q = np.empty((n, n), order="F") if cfg.accumulate_q else None
    fo, arrs = (_factors.alloc_host(n, n, cfg.b, False) if return_factors
                else _factors.alloc_tau(n, False))
    st = _lib.BrStats()
    rc = _dev.run_traced(h, groups, lambda: lib.br_reduce_sym_band_host(
        h, n, cfg.w, cfg.b, depth, A.ctypes.data, n, band.ctypes.data, n,
        Q.ctypes.data if Q is not None else None, n, fo, st))
    _lib.check(rc, "reduce_sym_band")
    variant = {SevpVariant.REFERENCE: "reference", SevpVariant.V1: "v1", SevpVariant.V2: "v2"}[cfg.variant]
    flops, iters = sevp_counted_flops(n, cfg.w, cfg.b, variant, cfg.accumulate_q, cfg.inner_b)
    apply_correction(flops, tau_zero_correction(_factors.sevp_panels(n, cfg.w, cfg.b), arrs["taul"],
                                                cfg.inner_b))
    for key, val in flops.items():
        if key != "total":
            FLOPS.add(key, val)
    if stats is not None:
        stats.update(device_ms=st.device_ms, launches=st.launches, iterations=st.iterations)
    fac = None
    if return_factors:
        fac = _factors.BandFactors(left=_factors.ChainFactors(
            arrs["yl"], arrs["tl"], arrs["taul"], _factors.sevp_panels(n, cfg.w, cfg.b), n))
    return SevpResult(band=band, q=Q, flops=flops, iterations=int(st.iterations), factors=fac)


def _reduce_multi(A, cfg, depth, devs, return_factors, stats):
    """reduce_sym_band over several GPUs (block-cyclic driver, multi.py)."""
    if cfg.accumulate_q or return_factors:
        raise ValueError("accumulate_q / return_factors are single-GPU features "
                         "(the block-cyclic driver does not keep Q or the factors)")
    _multi.check_dist_shape(cfg.n, cfg.w, cfg.b, "reduce_sym_band")
    n = cfg.n
    band, its, (taul, _) = _multi.reduce_devices(A, "sevp", cfg.w, cfg.b, devs, depth)
    variant = {SevpVariant.REFERENCE: "reference", SevpVariant.V1: "v1", SevpVariant.V2: "v2"}[cfg.variant]
    flops, _ = sevp_counted_flops(n, cfg.w, cfg.b, variant, False, cfg.inner_b)
    apply_correction(flops, tau_zero_correction(_factors.sevp_panels(n, cfg.w, cfg.b), taul,
                                                cfg.inner_b))
    for key, val in flops.items():
        if key != "total":
            FLOPS.add(key, val)
    if stats is not None:
        stats.update(iterations=its, devices=list(devs))
    return SevpResult(band=band, q=None, flops=flops, iterations=int(its))
