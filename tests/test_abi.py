"""The C-ABI library loads and exports every symbol include/bgs.h declares (CPU, no compute)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bgs.h")
LIB = os.path.join(ROOT, "paper_2605_13794_b200", "libbgs.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s*(bgs_[a-z_]+)\s*\(", src, re.M)))


def _lib():
    if not os.path.exists(LIB):
        from paper_2605_13794_b200.build import build
        build()
    return C.CDLL(LIB)


def test_header_declares_the_north_star_calls():
    fns = declared_functions()
    for name in ("bgs_project", "bgs_route", "bgs_sort_tiles", "bgs_raster_fwd", "bgs_raster_bwd", "bgs_importance",
                 "bgs_route_reverse", "bgs_project_bwd", "bgs_ctx_create", "bgs_last_error"):
        assert name in fns


def test_library_exports_every_declared_symbol():
    lib = _lib()
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    import paper_2605_13794_b200.bgs as B
    assert set(declared_functions()) <= set(B.EXPORTS)


def test_no_cpu_fallback_without_device():
    """Without a CUDA device the library refuses instead of computing on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2605_13794_b200.bgs as B
    with pytest.raises(B.BgsError) as e:
        B.Context()
    assert "BGS_ERR_CUDA" in str(e.value)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2605_13794_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower().replace("oracle's", ""), f
