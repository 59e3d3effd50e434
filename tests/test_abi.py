"""The C-ABI library (include/hgs.h) loads and exports every declared
symbol; the Python bindings cover exactly the declared API.  CPU only: no
compute call is made."""

import ctypes
import os
import re

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "hgs.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w]+\s*\*?\s*(hgs_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_operator_surface():
    names = declared_functions()
    for n in ("hgs_preprocess", "hgs_build_tiles", "hgs_blend_forward", "hgs_blend_backward", "hgs_project_backward",
              "hgs_rasterize_fragments", "hgs_sample_texture", "hgs_texture_backward", "hgs_composite_loss",
              "hgs_transmittance_mask", "hgs_adam_step", "hgs_last_error"):
        assert n in names, n


def test_library_exports_every_declared_symbol():
    from paper_2506_06988_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, f"libhgs.so lacks {missing}"
    assert set(declared_functions()) == set(_lib.SIGNATURES), "Python bindings out of sync with include/hgs.h"
    assert _lib.load().hgs_abi_version() == 1


def test_argument_errors_map_to_value_error():
    from paper_2506_06988_b200 import _lib
    lib = _lib.load()
    # NULL arguments are rejected before any CUDA call
    st = lib.hgs_transmittance_mask(None, 10, 20.0, 0, None, None)
    assert st == _lib.HGS_ERR_INVALID
    with pytest.raises(ValueError):
        _lib.check(st, "hgs_transmittance_mask")
    assert lib.hgs_transmittance_mask(None, 10, 20.0, 9, None, None) == _lib.HGS_ERR_INVALID
    assert b"null" in lib.hgs_last_error() or b"variant" in lib.hgs_last_error()


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2506_06988_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert not re.search(r"^\s*(from|import)\s+[\w.]*oracle", src, flags=re.M), fn
            assert "liboracle" not in src and "gsmesh_oracle" not in src, fn
