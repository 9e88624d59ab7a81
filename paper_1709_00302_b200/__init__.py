"""B200-native (sm_100a) first-stage band reduction, arXiv 1709.00302.

Drop-in for the reference package `bandred`'s hot path: the same public
names, arguments, result types and error behaviour, with the arithmetic in
hand-written CUDA (libbandred_b200.so, C ABI in include/bandred_b200.h).

    import paper_1709_00302_b200 as bandred
    res = bandred.reduce_sym_band(A, bandred.SevpConfig(n, w, b, bandred.SevpVariant.V2))

There is no CPU fallback: every compute entry point raises if the CUDA
library or device is missing.
"""
from .checks import band_check, orth_residual, spectra_match
from .cli import gen_general, gen_sym, load_matrix, save_matrix
from .flops import FLOPS, FlopCounter, reset_flops, snapshot_flops, sevp_nominal_flops, svd_nominal_flops
from .kernels import (
    PanelFactors,
    apply_wy_left,
    apply_wy_right,
    build_w,
    house_gen,
    lq_panel,
    qr_panel,
    sym_two_sided_update,
    symm_lower,
    syr2k_lower,
)
from .runtime import EventTrace, ExecGroups, WriteOverlapError
from .sevp import SevpConfig, SevpResult, SevpVariant, V2Mapping, reduce_sym_band
from .svd import SvdConfig, SvdForm, SvdResult, SvdVariant, reduce_band_svd, reduce_tri_band
from .stage2 import band_to_bidiagonal, band_to_tridiagonal
from ._dev import set_device, get_device

__all__ = [
    "FLOPS",
    "FlopCounter",
    "reset_flops",
    "snapshot_flops",
    "PanelFactors",
    "house_gen",
    "qr_panel",
    "lq_panel",
    "build_w",
    "apply_wy_left",
    "apply_wy_right",
    "symm_lower",
    "syr2k_lower",
    "sym_two_sided_update",
    "ExecGroups",
    "EventTrace",
    "WriteOverlapError",
    "SevpConfig",
    "SevpResult",
    "SevpVariant",
    "V2Mapping",
    "reduce_sym_band",
    "sevp_nominal_flops",
    "SvdConfig",
    "SvdResult",
    "SvdForm",
    "SvdVariant",
    "reduce_tri_band",
    "reduce_band_svd",
    "svd_nominal_flops",
    "band_to_tridiagonal",
    "band_to_bidiagonal",
    "band_check",
    "orth_residual",
    "spectra_match",
    "gen_general",
    "gen_sym",
    "save_matrix",
    "load_matrix",
    "set_device",
    "get_device",
]

__version__ = "0.1.0"
