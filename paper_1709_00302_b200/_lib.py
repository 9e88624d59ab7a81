"""ctypes binding of the C ABI in include/bandred_b200.h.

The shared library is built in-tree (paper_1709_00302_b200/_lib/) by
`paper_1709_00302_b200.build`. There is no CPU fallback: if the library is
missing or no CUDA device is present, every GPU entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libbandred_b200.so")

i64 = C.c_int64
dptr = C.c_void_p


class BrStats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64),
        ("device_ms", C.c_double),
        ("nominal_flops", C.c_double),
        ("launches", C.c_int64),
    ]


class BrFactors(C.Structure):
    """br_factors (include/bandred_b200.h): packed per-panel Y / T / tau."""
    _fields_ = [
        ("yl", C.c_void_p), ("ldyl", C.c_int64), ("tl", C.c_void_p), ("ldtl", C.c_int64),
        ("taul", C.c_void_p),
        ("yr", C.c_void_p), ("ldyr", C.c_int64), ("tr", C.c_void_p), ("ldtr", C.c_int64),
        ("taur", C.c_void_p),
    ]


BR_OPT_MAX_ITERS = 1

# name -> (restype, argtypes); mirrors include/bandred_b200.h exactly
SIGNATURES = {
    "br_version": (C.c_int, []),
    "br_last_error": (C.c_char_p, []),
    "br_launch_count": (C.c_int64, []),
    "br_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "br_destroy": (C.c_int, [C.c_void_p]),
    "br_set_streams": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "br_sync": (C.c_int, [C.c_void_p]),
    "br_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "br_get_timing": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_int64)]),
    "br_stream_select": (C.c_int, [C.c_void_p, C.c_int]),
    "br_stream_join": (C.c_int, [C.c_void_p, C.c_int]),
    "br_gemm": (C.c_int, [C.c_void_p, C.c_int, C.c_int, i64, i64, i64, C.c_double, dptr, i64, dptr,
                          i64, C.c_double, dptr, i64]),
    "br_symm_lower_ex": (C.c_int, [C.c_void_p, i64, i64, C.c_double, dptr, i64, dptr, i64,
                                   C.c_double, dptr, i64]),
    "br_house_gen": (C.c_int, [C.c_void_p, i64, dptr, dptr, dptr]),
    "br_qr_panel": (C.c_int, [C.c_void_p, i64, i64, dptr, i64, dptr, i64, dptr, i64, dptr, i64, dptr]),
    "br_lq_panel": (C.c_int, [C.c_void_p, i64, i64, dptr, i64, dptr, i64, dptr, i64, dptr, i64, dptr]),
    "br_build_w": (C.c_int, [C.c_void_p, i64, i64, dptr, i64, dptr, i64, dptr, i64]),
    "br_apply_wy_left": (C.c_int, [C.c_void_p, i64, i64, dptr, i64, dptr, i64, dptr, i64, i64]),
    "br_apply_wy_right": (C.c_int, [C.c_void_p, i64, i64, dptr, i64, dptr, i64, dptr, i64, i64]),
    "br_symm_lower": (C.c_int, [C.c_void_p, i64, i64, dptr, i64, dptr, i64, dptr, i64]),
    "br_syr2k_lower": (C.c_int, [C.c_void_p, i64, i64, dptr, i64, dptr, i64, dptr, i64, i64, i64]),
    "br_symm_lower_cyclic": (C.c_int, [C.c_void_p, i64, i64, i64, dptr, i64, dptr, i64, dptr, i64,
                                       i64, i64, i64, i64, i64]),
    "br_syr2k_lower_cyclic": (C.c_int, [C.c_void_p, i64, i64, i64, dptr, i64, dptr, i64, dptr, i64,
                                        i64, i64, i64]),
    "br_band_to_tridiag": (C.c_int, [C.c_void_p, i64, i64, dptr, i64, dptr, dptr]),
    "br_band_to_bidiag": (C.c_int, [C.c_void_p, i64, i64, i64, dptr, i64, dptr, dptr]),
    "br_sym_two_sided_update": (C.c_int, [C.c_void_p, i64, i64, dptr, i64, dptr, i64, dptr, i64]),
    "br_set_option": (C.c_int, [C.c_void_p, C.c_int, i64]),
    "br_reduce_sym_band": (C.c_int, [C.c_void_p, i64, i64, i64, C.c_int, dptr, i64, dptr, i64,
                                     C.POINTER(BrFactors), C.POINTER(BrStats)]),
    "br_reduce_tri_band": (C.c_int, [C.c_void_p, i64, i64, i64, i64, C.c_int, dptr, i64,
                                     C.POINTER(BrFactors), C.POINTER(BrStats)]),
    "br_sym_stage_bytes": (C.c_int64, [i64]),
    "br_reduce_sym_band_host": (C.c_int, [C.c_void_p, i64, i64, i64, C.c_int, dptr, i64, dptr, i64,
                                          dptr, i64, C.POINTER(BrFactors), C.POINTER(BrStats)]),
    "br_reduce_tri_band_host": (C.c_int, [C.c_void_p, i64, i64, i64, i64, C.c_int, dptr, i64, dptr,
                                          i64, C.POINTER(BrFactors), C.POINTER(BrStats)]),
    "br_trace_count": (i64, [C.c_void_p]),
    "br_trace_get": (C.c_int, [C.c_void_p, i64, C.c_char_p, i64, C.POINTER(C.c_int),
                               C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "br_reduce_band": (C.c_int, [C.c_void_p, i64, i64, i64, i64, C.c_int, C.c_int, dptr, i64,
                                 C.POINTER(BrFactors), C.POINTER(BrStats)]),
    "br_reduce_band_host": (C.c_int, [C.c_void_p, i64, i64, i64, i64, C.c_int, C.c_int, dptr, i64,
                                      dptr, i64, C.POINTER(BrFactors), C.POINTER(BrStats)]),
}

_lib = None
_lock = threading.Lock()
_handles: dict[int, int] = {}


class BandredError(RuntimeError):
    """A CUDA failure inside the library (positive status code)."""


def load(path: str | None = None):
    """Load (once) and return the ctypes library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise RuntimeError(
                f"CUDA library {p} not built; run `python -m paper_1709_00302_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = C.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int, what: str):
    if rc == 0:
        return
    msg = load().br_last_error().decode(errors="replace")
    if rc < 0:
        raise ValueError(f"{what}: {msg}")
    raise BandredError(f"{what} failed (status {rc}): {msg}")


def handle(device: int = 0) -> int:
    """Per-device context (streams, workspace), created on first use."""
    lib = load()
    with _lock:
        h = _handles.get(device)
        if h is None:
            out = C.c_void_p()
            rc = lib.br_create(device, C.byref(out))
            if rc != 0:
                msg = lib.br_last_error().decode(errors="replace")
                raise BandredError(f"br_create(device={device}) failed ({rc}): {msg}")
            h = out.value
            _handles[device] = h
        return h
