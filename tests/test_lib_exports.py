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


def test_cooperative_launch_refusal_is_recognised():
    """A refused cooperative launch (nothing ran) hands over to the multi-launch path with a
    warning; a barrier timeout (CL_EARG + 1) or a fault is not treated as a refusal."""
    import warnings
    from paper_2407_15049_b200 import _lib
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        assert _lib.coop_refused(720, "cl_admm_step_diag_fused")
        assert not _lib.coop_refused(0, "x") and not _lib.coop_refused(_lib.CL_EARG + 1, "x")
        assert not _lib.coop_refused(700, "x")          # an illegal address is a fault, not a refusal
    assert len(w) == 1 and "multi-launch" in str(w[0].message)


def test_inconsistent_arguments_return_earg_without_device():
    """Argument checks run before any device work: inconsistent sizes or missing operands
    return CL_EARG (the header's error contract), on a host with no GPU as on a B200."""
    import ctypes as C
    from paper_2407_15049_b200 import _lib, build_ext
    build_ext.build()
    lib = _lib.load(require_device=False)
    E = _lib.CL_EARG
    assert lib.cl_lincomb(None, 10, None, None, None) == E                     # no args
    a = _lib.LincombArgs()
    a.nin = _lib.CL_MAXIN + 1
    assert lib.cl_lincomb(C.byref(a), 10, None, None, None) == E               # too many inputs
    assert lib.cl_pattern_spmm(None, None, 26, 1.0, None, None, None, None, None) == E
    s = _lib.Pattern()
    assert lib.cl_pattern_spmm(C.byref(s), None, 26, 1.0, None, None, None, None, None) == E
    assert lib.cl_gather_rows(None, -1, 26, None, None, None) == E             # negative count
    assert lib.cl_gather_rows(None, 5, 26, None, None, None) == E              # missing operands
    assert lib.cl_gather_rows(None, 0, 26, None, None, None) == 0              # empty is fine
