"""The C-ABI library loads and exports every symbol include/culorads.h declares (CPU)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "culorads.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(cl_[a-z_0-9]+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "cl_lincomb" in syms and "cl_pattern_spmm" in syms and "cl_constraint_eval" in syms


def test_library_exports_all_declared_symbols():
    from paper_2407_15049_b200 import _lib, build_ext
    build_ext.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(_lib.EXPORTS) == set(declared_symbols())
    lib.cl_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.cl_version()


def test_no_cpu_fallback_without_device():
    import torch
    from paper_2407_15049_b200 import _lib
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(_lib.CulLoradsError):
        _lib.load(require_device=True)
