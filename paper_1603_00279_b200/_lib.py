"""ctypes declarations of the C-ABI in include/tsf.h (argument marshalling only).

The shared library is built in-tree (paper_1603_00279_b200/lib/libtsf.so).  There is no
fallback: if the library is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TSF_LIB_VARIANT=<name> selects a developer build lib/libtsf_<name>.so (e.g. "prof", the
# section-timer build); unset = the product library
_VARIANT = os.environ.get("TSF_LIB_VARIANT", "")
LIB_PATH = os.path.join(HERE, "lib", f"libtsf_{_VARIANT}.so" if _VARIANT else "libtsf.so")

TSF_OK = 0
TSF_W_MAXIT = 1
ERRORS = {-1: "TSF_E_ARG", -2: "TSF_E_WORKSPACE", -3: "TSF_E_CUDA", -4: "TSF_E_SINGULAR_PREC",
          -5: "TSF_E_BREAKDOWN", -6: "TSF_E_DIVERGED", -7: "TSF_E_STATE"}
BICGSTAB, CGNR, PCGS, GSF = 0, 1, 2, 3
STRANG, TCHAN, NOPREC = 0, 1, 2
SRC_ZERO, SRC_SEPARABLE, SRC_TABLE, SRC_CALLBACK = 0, 1, 2, 3

FN_T = C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p)
SRC_CB = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.c_int64, C.c_double, C.POINTER(C.c_double), C.c_void_p)
PD = C.POINTER(C.c_double)


class TsfProblem(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("n", C.c_int64), ("M", C.c_int64),
                ("a", C.c_double), ("b", C.c_double), ("T", C.c_double),
                ("gamma_t", PD), ("dplus_t", PD), ("dminus_t", PD),
                ("gamma_fn", FN_T), ("dplus_fn", FN_T), ("dminus_fn", FN_T), ("coef_ctx", C.c_void_p),
                ("phi", PD), ("phi_fn", FN_T), ("phi_ctx", C.c_void_p),
                ("src_kind", C.c_int32), ("K", C.c_int32),
                ("basis", PD), ("scal", PD), ("f_table", PD), ("f_table_on_device", C.c_int32),
                ("f_cb", SRC_CB), ("f_ctx", C.c_void_p)]


class TsfSolver(C.Structure):
    _fields_ = [("method", C.c_int32), ("precond", C.c_int32), ("tol", C.c_double),
                ("maxit", C.c_int32), ("cluster", C.c_int32), ("x0_warm", C.c_int32),
                ("true_residual", C.c_int32), ("pipelined", C.c_int32),
                ("hist_block", C.c_int32)]


class TsfPlanInfo(C.Structure):
    _fields_ = [("cluster", C.c_int32), ("threads", C.c_int32), ("smem_bytes", C.c_int64),
                ("embed_len", C.c_int64), ("precond_len", C.c_int64),
                ("workspace_bytes", C.c_size_t), ("exchange", C.c_int32), ("chunk", C.c_int32),
                ("vsmem", C.c_int32), ("resident", C.c_int32)]


class TsfError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where}: {ERRORS.get(code, code)}: {msg}")
        self.code = code


_lib = None

_SIGS = {
    "tsf_sample_points": (C.c_int, [C.POINTER(TsfProblem), PD, PD]),
    "tsf_plan": (C.c_int, [C.POINTER(TsfProblem), C.c_int32, C.POINTER(TsfSolver), C.POINTER(TsfPlanInfo)]),
    "tsf_workspace_bytes": (C.c_int, [C.POINTER(TsfProblem), C.c_int32, C.POINTER(TsfSolver),
                                      C.POINTER(C.c_size_t)]),
    "tsf_init": (C.c_int, [C.POINTER(TsfProblem), C.c_int32, C.POINTER(TsfSolver), C.c_void_p,
                           C.c_size_t, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "tsf_step": (C.c_int, [C.c_void_p]),
    "tsf_solve": (C.c_int, [C.c_void_p]),
    "tsf_reset": (C.c_int, [C.c_void_p]),
    "tsf_sync": (C.c_int, [C.c_void_p]),
    "tsf_level": (C.c_int64, [C.c_void_p]),
    "tsf_get_solution": (C.c_int, [C.c_void_p, C.c_int32, PD, C.c_int32]),
    "tsf_get_solutions": (C.c_int, [C.c_void_p, PD, C.c_int32]),
    "tsf_get_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), PD, C.POINTER(C.c_int32)]),
    "tsf_get_true_residuals": (C.c_int, [C.c_void_p, PD]),
    "tsf_handle_info": (C.c_int, [C.c_void_p, C.POINTER(TsfPlanInfo)]),
    "tsf_destroy": (C.c_int, [C.c_void_p]),
    "tsf_last_error": (C.c_char_p, []),
    "tsf_debug_fft_tables": (C.c_int, [C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "tsf_debug_local_fft": (C.c_int, [C.c_int64, PD, PD, C.c_int32]),
    "tsf_debug_weights": (C.c_int, [C.c_double, C.c_int64, PD, PD]),
    "tsf_debug_apply": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, PD, PD]),
    "tsf_debug_apply_bench": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.POINTER(C.c_float)]),
    "tsf_debug_spectra": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, PD, PD]),
    "tsf_debug_rhs": (C.c_int, [C.c_void_p, C.c_int32, PD]),
    "tsf_debug_set_history": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, PD]),
    "tsf_debug_prof": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.c_int32]),
    "tsf_debug_helper_state": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
}

EXPORTED = tuple(_SIGS)


def load():
    """Load libtsf.so (raises if it is missing: there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (nvcc, sm_100a)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if _VARIANT and not hasattr(lib, name):
                continue          # developer variants (e.g. an older build) may lack new hooks
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, where: str) -> int:
    if rc < 0:
        msg = load().tsf_last_error()
        raise TsfError(rc, where, msg.decode() if msg else "")
    return rc
