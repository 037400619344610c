"""ctypes binding of libculorads (include/culorads.h).

The shared library is built in-tree by ``paper_2407_15049_b200.build_ext``
(``nvcc -gencode arch=compute_100a,code=sm_100a``). There is no fallback:
if the library or an sm_100 device is missing, ``lib()`` raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CULORADS_LIB") or os.path.join(HERE, "libculorads.so")

CL_MAXIN = 20
CL_MAXDOT = 48
CL_MAXY = 4
CL_RED_BLOCKS = 1184
CL_WS_DOUBLES = CL_RED_BLOCKS * CL_MAXDOT
CL_WS_ALLOC = CL_WS_DOUBLES + 8
CL_OUT = 255
CL_DOT_PAIRS, CL_DOT_OUT_ALL, CL_DOT_FIRST_TWO = 0, 1, 2
CL_EARG = 1001
# cudaError codes with which a cooperative launch is refused before anything runs
# (LaunchOutOfResources, CooperativeLaunchTooLarge, NotPermitted, NotSupported): the
# one-launch paths then give way to the multi-launch ones
COOP_REFUSED = (701, 720, 800, 801)


def coop_refused(rc, what):
    """True (with a one-time warning) when a cooperative launch was refused."""
    if rc not in COOP_REFUSED:
        return False
    import warnings
    warnings.warn(f"{what}: cooperative launch refused (cudaError {rc}); using the multi-launch path",
                  RuntimeWarning, stacklevel=3)
    return True


CL_EBARRIER = CL_EARG + 1    # a one-launch kernel's grid barrier timed out (its state was reset)


def barrier_timeout(rc, what):
    """True (with a warning) when a one-launch kernel's grid barrier gave up (about 1 s of
    waiting: GPU time-slicing, MPS or a debugger). Its outputs are void; the caller reruns
    the work on the multi-launch path from the inputs it kept."""
    if rc != CL_EBARRIER:
        return False
    import warnings
    warnings.warn(f"{what}: grid barrier timed out; rerunning on the multi-launch path",
                  RuntimeWarning, stacklevel=3)
    return True

EXPORTS = ("cl_lincomb", "cl_pattern_spmm", "cl_constraint_eval", "cl_constraint_eval_halo", "cl_constraint_eval_pair",
           "cl_diag_constraint_eval", "cl_sddmm",
           "cl_gather_rows", "cl_diag_cg_apply", "cl_diag_cg_apply_rows", "cl_diag_cg_step", "cl_cg_step", "cl_cg_step_dev", "cl_admm_step_diag", "cl_admm_step_diag_fused", "cl_admm_step_generic", "cl_alm_inner_diag", "cl_alm_inner_diag_fused", "cl_alm_inner_generic",
           "cl_diag_admm_cg_init", "cl_diag_admm_step_end", "cl_diag_admm_step_end_rows", "cl_single_entry_apply", "cl_single_entry_apply_pair", "cl_pair_pack", "cl_cg_direction_pair", "cl_lanczos_loop", "cl_lanczos_loop_fused",
           "cl_pattern_assemble", "cl_lanczos_update",
           "cl_diag_alm_update", "cl_basis_project", "cl_basis_subtract",
           "cl_set_l2_fetch_granularity", "cl_get_l2_fetch_granularity", "cl_ipc_export", "cl_ipc_import",
           "cl_ipc_close", "cl_version", "cl_device_ok")

CL_IPC_HANDLE_BYTES = 64
CL_MAX_PEERS = 8
CL_GHOST_PEERS = -2

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
D = ctypes.c_double


class LincombArgs(ctypes.Structure):
    _fields_ = [("nin", I32), ("mode", I32), ("ndot", I32),
                ("inp", P * CL_MAXIN), ("coef", D * CL_MAXIN), ("out", P),
                ("da", ctypes.c_uint8 * CL_MAXDOT), ("db", ctypes.c_uint8 * CL_MAXDOT)]


class Pattern(ctypes.Structure):
    _fields_ = [("nrows", I64), ("indptr", P), ("indices", P), ("cv", P), ("c_coeff", D),
                ("at_ptr", P), ("at_con", P), ("at_val", P), ("w1", P), ("w2", P),
                ("nnz", I64), ("scratch", P), ("ghost", P), ("nown", I64),
                ("w1g", P), ("w2g", P), ("mown", I64)]


class Epilogue(ctypes.Structure):
    _fields_ = [("ny", I32), ("Y", P * CL_MAXY), ("ycoef", D * CL_MAXY),
                ("nz", I32), ("Z", P * CL_MAXY),
                ("ndot", I32), ("da", ctypes.c_uint8 * 8), ("db", ctypes.c_uint8 * 8),
                ("drow", P), ("dmul", P)]


class DiagUpdateArgs(ctypes.Structure):
    _fields_ = [("n", I64), ("ld", I32), ("aval", P), ("tau", D), ("rho", D), ("scale", D),
                ("R", P), ("D", P), ("CR", P), ("CD", P),
                ("ax", P), ("ax_out", P), ("q1", P), ("q2", P),
                ("lam", P), ("b", P), ("g_old", P), ("g_new", P), ("y", P),
                ("nh", I32), ("H", P * CL_MAXIN), ("refresh", I32)]


EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32)
REDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                             ctypes.c_void_p)


RELEASE_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p)


class DistHooks(ctypes.Structure):
    _fields_ = [("ctx", P), ("exchange", EXCHANGE_FN), ("reduce", REDUCE_FN), ("nown", I64),
                ("release", RELEASE_FN)]


class AdmmDiagArgs(ctypes.Structure):
    _fields_ = [("n", I64), ("ld", I32), ("aval", P), ("b", P), ("lam", P), ("lam_new", P), ("ax", P),
                ("ax_valid", I32),
                ("pnorm2_known", D), ("U", P), ("V", P), ("U_new", P), ("V_new", P),
                ("r", P), ("r_v", P), ("p", P), ("Q", P), ("cu", P), ("nlam", P), ("res", P),
                ("cpat", Pattern), ("rho", D), ("scale", D), ("binf", D), ("rel_floor", D),
                ("primal_coeff", D), ("cg_cap", I32), ("slab", P), ("host", P), ("ws", P), ("stream", P),
                ("want_balance", I32), ("dist", ctypes.POINTER(DistHooks))]


class AdmmGenericArgs(ctypes.Structure):
    _fields_ = [("n", I64), ("m", I64), ("ld", I32), ("b", P), ("lam", P), ("ax", P), ("ax_new", P),
                ("U", P), ("V", P), ("U_new", P), ("V_new", P), ("rhs", P), ("r", P), ("p", P), ("Q", P),
                ("y", P), ("nlam", P), ("rhob", P), ("pair", P), ("con_indptr", P), ("con_pi", P), ("con_pj", P),
                ("con_val", P), ("omega", Pattern), ("apat", Pattern), ("single_a", P), ("rho", D), ("scale", D),
                ("binf", D), ("rel_floor", D), ("primal_coeff", D), ("cg_cap", I32), ("slab", P), ("host", P),
                ("ws", P), ("stream", P)]


class AdmmStepStats(ctypes.Structure):
    _fields_ = [("it_u", I32), ("it_v", I32), ("res_u", D), ("res_v", D), ("eps_u", D), ("eps_v", D),
                ("pnorm2", D), ("hit_cap", I32), ("status", I32), ("bad_half", I32), ("bad_is_new", I32),
                ("pq_bad", D), ("u_reused", I32), ("v_reused", I32), ("objective", D), ("lam_b", D),
                ("err_line", I32), ("du2", D), ("dv2", D)]


CL_ALM_MAXMEM = 8
CL_ALM_MAXBUF = 2 * CL_ALM_MAXMEM + 4


class AlmInnerArgs(ctypes.Structure):
    _fields_ = [("n", I64), ("ld", I32), ("memory", I32), ("max_iter", I32), ("tol", D), ("reduce_factor", D),
                ("rho", D), ("scale", D), ("b1", D), ("aval", P), ("b", P), ("lam", P), ("R", P), ("CR", P),
                ("CD", P), ("ax", P), ("ax2", P), ("q1", P), ("q2", P), ("wv", P), ("zero_g", P),
                ("nbuf", I32), ("bufs", P * CL_ALM_MAXBUF), ("cpat", Pattern), ("slab", P), ("host", P),
                ("ws", P), ("stream", P), ("rec_cap", I32), ("rec", P), ("gnorms", P),
                ("dist", ctypes.POINTER(DistHooks)), ("m", I64), ("con_indptr", P), ("con_pi", P), ("con_pj", P),
                ("con_val", P), ("apat", Pattern), ("res", P), ("pair", P)]


class AlmInnerStats(ctypes.Structure):
    _fields_ = [("iterations", I32), ("n_records", I32), ("n_gnorms", I32), ("hit_cap", I32), ("status", I32),
                ("ax_is_ax2", I32), ("err_line", I32)]


class LanczosArgs(ctypes.Structure):
    _fields_ = [("n", I64), ("k_max", I32), ("breakdown", D), ("Q", P), ("ldq", I64), ("u", P), ("r", P),
                ("h", P), ("S", Pattern), ("slab", P), ("host", P), ("ws", P), ("stream", P),
                ("alphas", P), ("betas", P), ("dbeta", P), ("dalpha", P)]


_LIB = None
_LOCK = threading.Lock()


class CulLoradsError(RuntimeError):
    pass


def _declare(lib):
    lib.cl_lincomb.argtypes = [ctypes.POINTER(LincombArgs), I64, P, P, P]
    lib.cl_pattern_spmm.argtypes = [ctypes.POINTER(Pattern), P, I32, D, ctypes.POINTER(Epilogue),
                                    P, P, P, P]
    lib.cl_constraint_eval.argtypes = [I64, P, P, P, P, I32, P, P, P, P, P, P, P, P, P]
    lib.cl_constraint_eval_halo.argtypes = [I64, P, P, P, P, I32, P, P, P, P, P, P, P, P, P, I64, P]
    lib.cl_constraint_eval_pair.argtypes = [I64, P, P, P, P, I32, P, P, P, P]
    lib.cl_diag_constraint_eval.argtypes = [I64, P, I32, P, P, P, P, P, P, P, P, P]
    lib.cl_diag_cg_apply.argtypes = [I64, I32, P, D, D, P, P, P, P, P, P, P]
    lib.cl_cg_step.argtypes = [I64, D, P, P, P, P, P, P, P, P]
    lib.cl_diag_cg_apply_rows.argtypes = [I64, I32, P, D, D, P, P, P, P, P, P, P]
    lib.cl_diag_cg_step.argtypes = [I64, I32, D, P, P, D, D, P, P, P, P, P, P, P, P]
    lib.cl_admm_step_diag.argtypes = [ctypes.POINTER(AdmmDiagArgs), ctypes.POINTER(AdmmStepStats)]
    lib.cl_admm_step_diag_fused.argtypes = [ctypes.POINTER(AdmmDiagArgs), ctypes.POINTER(AdmmStepStats)]
    lib.cl_admm_step_generic.argtypes = [ctypes.POINTER(AdmmGenericArgs), ctypes.POINTER(AdmmStepStats)]
    lib.cl_alm_inner_diag.argtypes = [ctypes.POINTER(AlmInnerArgs), ctypes.POINTER(AlmInnerStats)]
    lib.cl_alm_inner_diag_fused.argtypes = [ctypes.POINTER(AlmInnerArgs), ctypes.POINTER(AlmInnerStats)]
    lib.cl_alm_inner_generic.argtypes = [ctypes.POINTER(AlmInnerArgs), ctypes.POINTER(AlmInnerStats)]
    lib.cl_diag_admm_cg_init.argtypes = [ctypes.POINTER(Pattern), P, P, I32, D, D, P, P, P, P, P, P, P]
    lib.cl_diag_admm_step_end_rows.argtypes = [I64, I32, P, P, P, P, P, P, D, P, P, P, P, P]
    lib.cl_diag_admm_step_end.argtypes = [ctypes.POINTER(Pattern), P, P, I32, P, P, P, D, P, P, P, P, P]
    lib.cl_single_entry_apply.argtypes = [I64, P, P, P, I32, P, P, D, P, P, P, P]
    lib.cl_single_entry_apply_pair.argtypes = [I64, P, P, P, I32, P, D, P, P, P, P]
    lib.cl_pair_pack.argtypes = [I64, I32, P, P, I32, P]
    lib.cl_cg_direction_pair.argtypes = [I64, I32, D, P, P, P, P]
    lib.cl_pattern_assemble.argtypes = [ctypes.POINTER(Pattern), P, P]
    lib.cl_lanczos_loop.argtypes = [ctypes.POINTER(LanczosArgs), ctypes.POINTER(I32)]
    lib.cl_lanczos_loop_fused.argtypes = [ctypes.POINTER(LanczosArgs), ctypes.POINTER(I32)]
    lib.cl_lanczos_update.argtypes = [I32, I64, P, P, P, P, P, P, P, P, P, P]
    lib.cl_cg_step_dev.argtypes = [I64, D, P, P, P, P, P, P, P, P, P]
    lib.cl_gather_rows.argtypes = [P, I64, I32, P, P, P]
    lib.cl_sddmm.argtypes = [I64, P, P, I32, P, P, P, P]
    lib.cl_diag_alm_update.argtypes = [ctypes.POINTER(DiagUpdateArgs), P, P, P]
    lib.cl_basis_project.argtypes = [P, I64, I32, I64, P, P, P, P]
    lib.cl_basis_subtract.argtypes = [P, I64, I32, I64, P, P, P]
    lib.cl_set_l2_fetch_granularity.argtypes = [I32]
    lib.cl_get_l2_fetch_granularity.argtypes = []
    lib.cl_ipc_export.argtypes = [P, P, ctypes.POINTER(I64)]
    lib.cl_ipc_import.argtypes = [P, ctypes.POINTER(P)]
    lib.cl_ipc_close.argtypes = [P]
    lib.cl_version.restype = ctypes.c_char_p
    lib.cl_device_ok.restype = ctypes.c_int
    for name in EXPORTS:
        if name not in ("cl_version", "cl_device_ok"):
            getattr(lib, name).restype = ctypes.c_int


def load(require_device=True):
    """Load (once) and return the library handle; raise loudly if unusable."""
    global _LIB
    with _LOCK:
        if _LIB is None:
            if not os.path.exists(LIB_PATH):
                raise CulLoradsError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -m paper_2407_15049_b200.build_ext` (no CPU fallback exists)")
            lib = ctypes.CDLL(LIB_PATH)
            _declare(lib)
            _LIB = lib
    if require_device and not _LIB.cl_device_ok():
        raise CulLoradsError("no sm_100 (B200) CUDA device visible; the solver has no CPU path")
    return _LIB


def check(rc, what):
    if rc != 0:
        raise CulLoradsError(f"{what} failed with code {rc}")
