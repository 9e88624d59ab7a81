"""The C-ABI library builds, loads and exports every symbol include/*.h
declares; the ctypes binding matches the header. CPU only (no compute)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bandred_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(br_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1709_00302_b200 import _lib
    from paper_1709_00302_b200 import build as b

    path = b.build()
    assert os.path.exists(path)
    return _lib.load(path)


def test_header_declares_the_reference_surface():
    names = header_functions()
    for want in ("br_qr_panel", "br_lq_panel", "br_build_w", "br_apply_wy_left", "br_apply_wy_right",
                 "br_symm_lower", "br_syr2k_lower", "br_sym_two_sided_update", "br_house_gen",
                 "br_reduce_sym_band", "br_reduce_tri_band", "br_reduce_sym_band_host",
                 "br_reduce_tri_band_host", "br_last_error", "br_create", "br_destroy"):
        assert want in names, want


def test_every_header_symbol_is_exported(lib):
    for name in header_functions():
        assert hasattr(lib, name), f"{name} missing from the shared library"


def test_ctypes_binding_matches_header(lib):
    from paper_1709_00302_b200 import _lib

    assert sorted(_lib.SIGNATURES) == header_functions()


def test_version_and_error_text(lib):
    assert lib.br_version() >= 100
    assert isinstance(lib.br_last_error(), bytes)


def test_sass_uses_fp64_tensor_cores_and_clusters():
    """The update kernels are DMMA (FP64 tensor core) code and the panel leaf
    uses DSMEM async stores; checked on the built sm_100a objects."""
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    obj = os.path.join(ROOT, "paper_1709_00302_b200", "_build")
    sass = subprocess.run([cuobjdump, "-sass", os.path.join(obj, "gemm_tile_C.o")],
                          capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass
    sass = subprocess.run([cuobjdump, "-sass", os.path.join(obj, "panel.o")],
                          capture_output=True, text=True).stdout
    assert "STAS" in sass and "SYNCS" in sass
