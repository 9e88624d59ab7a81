"""Dense general -> upper triangular-band on the B200 (drop-in for ref svd.py).

`reduce_tri_band(A, w, b, groups=None, range_log=None, inner_b=16)` keeps
the reference signature and semantics (ref svd.py:205-247): m < n reduces
A^T and transposes back (lower_bw = w, upper_bw = 0); off-band entries are
exactly 0. The reference schedule is strictly sequential; the GPU adds
look-ahead (keyword `lookahead`, default 1): the LQ panel and the next QR
panel are factored on the panel stream while the rank-b halves of the
left/right updates run. The split updates are bitwise identical to the
sequential order on the same GPU.

`reduce_band_svd(A, cfg)` dispatches cfg.form == TRIANGULAR_BAND to
reduce_tri_band exactly like ref svd.py:552-553 and runs the equal-bandwidth
BAND form (ref svd.py:250-589) on the GPU: REFERENCE / V1 apply the left
then the right trailing update, SIMULTANEOUS / V2 the fused two-sided
update; V1 / V2 add static look-ahead (both next panels factored on the
panel stream), bitwise equal to REFERENCE / SIMULTANEOUS on the same GPU.
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _dev, _lib
from . import factors as _factors
from . import multi as _multi
from .flops import (FLOPS, apply_correction, band_counted_flops, svd_nominal_flops,  # noqa: F401
                    tau_zero_correction, tri_counted_flops)
from .sevp import V2Mapping


class SvdForm(Enum):
    TRIANGULAR_BAND = "triband"
    BAND = "band"


class SvdVariant(Enum):
    REFERENCE = "reference"
    SIMULTANEOUS = "simultaneous"
    V1 = "v1"
    V2 = "v2"


@dataclass
class SvdConfig:
    m: int
    n: int
    w: int
    b: int
    form: SvdForm = SvdForm.BAND
    variant: SvdVariant = SvdVariant.REFERENCE
    v2_mapping: V2Mapping = V2Mapping.ON_TS
    inner_b: int = 16

    def validate(self):
        """Same rules and messages as ref svd.py:81-101."""
        if self.m < 1 or self.n < 1:
            raise ValueError("m, n >= 1")
        if self.w < 1:
            raise ValueError("w >= 1")
        if not (1 <= self.b <= self.w):
            raise ValueError("need 1 <= b <= w")
        if self.form == SvdForm.TRIANGULAR_BAND:
            if self.variant != SvdVariant.REFERENCE:
                raise ValueError("triangular-band form supports only the reference schedule")
        elif self.variant == SvdVariant.V1 and 2 * self.b > self.w:
            raise ValueError(f"V1 requires 2b <= w, got b={self.b}, w={self.w}")
        elif self.variant == SvdVariant.V2 and 2 * self.b <= self.w:
            warnings.warn(
                f"V2 with 2b <= w (b={self.b}, w={self.w}) is valid but outside "
                "its intended regime; V1 covers this case",
                RuntimeWarning,
                stacklevel=3,
            )


@dataclass
class SvdResult:
    band: np.ndarray
    flops: dict
    form: SvdForm
    lower_bw: int
    upper_bw: int
    iterations: int
    factors: "_factors.BandFactors | None" = None  # extension: return_factors=True


def _depth(groups, lookahead):
    if lookahead is not None:
        if lookahead not in (0, 1):
            raise ValueError("lookahead must be 0 or 1")
        return int(lookahead)
    if groups is not None and getattr(groups, "ts_count", 1) == 0:
        return 0
    return 1


def _swap(fac):
    # factors of A^T: its left chain is A's right chain and vice versa
    return None if fac is None else _factors.BandFactors(left=fac.right, right=fac.left)


def reduce_tri_band(A, w, b, groups=None, range_log=None, inner_b=16, *, lookahead=None,
                    device=None, stats=None, return_factors=False, ngpus=None, devices=None):
    """Reduce A to upper triangular-band form (band[i,j] = 0 for i > j or j > i + w).

    return_factors=True (extension) adds `factors`: the QR chain (left, U)
    and the LQ chain (right, V) with A = U B V^T (see factors.py).
    ngpus / devices (extension): the 1D block-cyclic multi-GPU
    driver over those devices from this one process (multi.py); square A,
    w == b, n a multiple of b, no factors."""
    if w < 1:
        raise ValueError("w >= 1")
    if not (1 <= b <= w):
        raise ValueError("need 1 <= b <= w")
    A = np.array(A, dtype=np.float64, order="F")
    if A.ndim != 2:
        raise ValueError("reduce_tri_band needs a 2-D matrix")
    if range_log is not None:
        raise ValueError("range_log instrumentation is a CPU-reference analysis feature; "
                         "not supported on the GPU path")
    depth = _depth(groups, lookahead)
    devs = _multi.resolve_devices(ngpus, devices)
    if devs is not None:
        return _reduce_tri_multi(A, w, b, inner_b, depth, devs, return_factors, stats)
    lib = _lib.load()
    h, _ = _dev.ctx(device)
    m, n = A.shape
    if m < n:
        inner = reduce_tri_band(np.asfortranarray(A.T), w, b, groups, None, inner_b,
                                lookahead=lookahead, device=device, stats=stats,
                                return_factors=return_factors)
        return SvdResult(band=np.asfortranarray(inner.band.T), flops=inner.flops,
                         form=SvdForm.TRIANGULAR_BAND, lower_bw=w, upper_bw=0,
                         iterations=inner.iterations, factors=_swap(inner.factors))
    band = np.empty((m, n), order="F")
    fo, arrs = _factors.alloc_host(m, n, b, True) if return_factors else _factors.alloc_tau(n, True)
    st = _lib.BrStats()
    rc = _dev.run_traced(h, groups, lambda: lib.br_reduce_tri_band_host(
        h, m, n, w, b, depth, A.ctypes.data, m, band.ctypes.data, m, fo, st))
    _lib.check(rc, "reduce_tri_band")
    flops, _ = tri_counted_flops(m, n, w, b, inner_b)
    pl, pr = _factors.tri_panels(m, n, w, b)
    apply_correction(flops, tau_zero_correction(pl, arrs["taul"], inner_b) +
                     tau_zero_correction(pr, arrs["taur"], inner_b))
    for key, val in flops.items():
        if key != "total":
            FLOPS.add(key, val)
    if stats is not None:
        stats.update(device_ms=st.device_ms, launches=st.launches, iterations=st.iterations)
    return SvdResult(band=band, flops=flops, form=SvdForm.TRIANGULAR_BAND, lower_bw=0, upper_bw=w,
                     iterations=int(st.iterations),
                     factors=_chains(arrs if return_factors else None, (pl, pr), m, n))


def _reduce_tri_multi(A, w, b, inner_b, depth, devs, return_factors, stats):
    """reduce_tri_band over several GPUs (block-cyclic driver, multi.py)."""
    m, n = A.shape
    if m != n:
        raise ValueError("reduce_tri_band on several GPUs needs a square matrix")
    if return_factors:
        raise ValueError("return_factors is a single-GPU feature (the block-cyclic driver "
                         "does not keep the factors)")
    _multi.check_dist_shape(n, w, b, "reduce_tri_band")
    band, its, (taul, taur) = _multi.reduce_devices(A, "tri", w, b, devs, depth)
    flops, _ = tri_counted_flops(m, n, w, b, inner_b)
    pl, pr = _factors.tri_panels(m, n, w, b)
    apply_correction(flops, tau_zero_correction(pl, taul, inner_b) +
                     tau_zero_correction(pr, taur, inner_b))
    for key, val in flops.items():
        if key != "total":
            FLOPS.add(key, val)
    if stats is not None:
        stats.update(iterations=its, devices=list(devs))
    return SvdResult(band=band, flops=flops, form=SvdForm.TRIANGULAR_BAND, lower_bw=0, upper_bw=w,
                     iterations=int(its))


def _chains(arrs, panels, m, n):
    if arrs is None:
        return None
    left, right = panels
    return _factors.BandFactors(
        left=_factors.ChainFactors(arrs["yl"], arrs["tl"], arrs["taul"], left, m),
        right=_factors.ChainFactors(arrs["yr"], arrs["tr"], arrs["taur"], right, n))


def reduce_band_svd(A, cfg, groups=None, range_log=None, *, lookahead=None, device=None,
                    stats=None, return_factors=False, ngpus=None, devices=None):
    """Dispatch on cfg.form (ref svd.py:515-589); m < n reduces A^T and swaps
    the bandwidth tags (ref svd.py:530-550); m <= w + 1 returns A unchanged.
    ngpus / devices: the triangular-band form only (multi.py)."""
    cfg.validate()
    multi = _multi.resolve_devices(ngpus, devices) is not None
    if multi and cfg.form != SvdForm.TRIANGULAR_BAND:
        raise ValueError("the band form has no multi-GPU driver; use form=TRIANGULAR_BAND")
    A = np.array(A, dtype=np.float64, order="F")
    if A.ndim != 2:
        raise ValueError("reduce_band_svd needs a 2-D matrix")
    if A.shape != (cfg.m, cfg.n):
        raise ValueError(f"cfg says {cfg.m} x {cfg.n} but the matrix is {A.shape[0]} x {A.shape[1]}")
    if cfg.m < cfg.n:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)  # already warned once
            tcfg = SvdConfig(m=cfg.n, n=cfg.m, w=cfg.w, b=cfg.b, form=cfg.form,
                             variant=cfg.variant, v2_mapping=cfg.v2_mapping, inner_b=cfg.inner_b)
            inner = reduce_band_svd(np.asfortranarray(A.T), tcfg, groups, range_log,
                                    lookahead=lookahead, device=device, stats=stats,
                                    return_factors=return_factors, ngpus=ngpus, devices=devices)
        return SvdResult(band=np.asfortranarray(inner.band.T), flops=inner.flops, form=cfg.form,
                         lower_bw=inner.upper_bw, upper_bw=inner.lower_bw,
                         iterations=inner.iterations, factors=_swap(inner.factors))
    if cfg.form == SvdForm.TRIANGULAR_BAND:
        return reduce_tri_band(A, cfg.w, cfg.b, groups, range_log, cfg.inner_b,
                               lookahead=lookahead, device=device, stats=stats,
                               return_factors=return_factors, ngpus=ngpus, devices=devices)
    if range_log is not None:
        if cfg.variant != SvdVariant.REFERENCE:
            raise ValueError("range logging is defined for the reference schedule")
        if cfg.w % cfg.b != 0:
            raise ValueError("range logging requires w to be a multiple of b")
        raise ValueError("range_log instrumentation is a CPU-reference analysis feature; "
                         "not supported on the GPU path")
    simultaneous = cfg.variant in (SvdVariant.SIMULTANEOUS, SvdVariant.V2)
    if lookahead is None:
        # V1 / V2 are the look-ahead schedules; REFERENCE / SIMULTANEOUS are
        # sequential (results are bitwise identical either way)
        lookahead = _depth(groups, None) if cfg.variant in (SvdVariant.V1, SvdVariant.V2) else 0
    depth = _depth(groups, lookahead)
    m, n, w, b = cfg.m, cfg.n, cfg.w, cfg.b
    lib = _lib.load()
    h, _ = _dev.ctx(device)
    band = np.empty((m, n), order="F")
    fo, arrs = _factors.alloc_host(m, n, b, True) if return_factors else _factors.alloc_tau(n, True)
    st = _lib.BrStats()
    rc = _dev.run_traced(h, groups, lambda: lib.br_reduce_band_host(
        h, m, n, w, b, int(simultaneous), depth, A.ctypes.data, m, band.ctypes.data, m, fo, st))
    _lib.check(rc, "reduce_band_svd")
    if st.iterations == 0:
        flops = {"total": 0}
    else:
        flops, _ = band_counted_flops(m, n, w, b, simultaneous, cfg.inner_b)
        pl, pr = _factors.band_panels(m, n, w, b)
        apply_correction(flops, tau_zero_correction(pl, arrs["taul"], cfg.inner_b) +
                         tau_zero_correction(pr, arrs["taur"], cfg.inner_b))
        for key, val in flops.items():
            if key != "total":
                FLOPS.add(key, val)
    if stats is not None:
        stats.update(device_ms=st.device_ms, launches=st.launches, iterations=st.iterations)
    return SvdResult(band=band, flops=flops, form=SvdForm.BAND, lower_bw=w, upper_bw=w,
                     iterations=int(st.iterations),
                     factors=_chains(arrs if return_factors else None, _factors.band_panels(m, n, w, b),
                                     m, n))
