"""ctypes declarations of the C ABI in include/bdfb.h (argument marshalling only).

Loads the in-tree paper_2405_01713_b200/libbdfb.so.  There is no fallback:
if the library is missing or does not load, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BDFB_LIB") or os.path.join(PKG, "libbdfb.so")   # BDFB_LIB: experiments only

MODEL_LINEAR, MODEL_ROBERTSON, MODEL_NYX_KWH, MODEL_MECH_H2, MODEL_MECH_DRM19, MODEL_MECH_GRI53 = 0, 1, 2, 3, 4, 5
LAYOUT_YC, LAYOUT_CY = 0, 1
MODE_PER_CELL, MODE_GLOBAL_NORM = 0, 1
KERNEL_AUTO, KERNEL_THREAD, KERNEL_GROUP, KERNEL_SPLIT = 0, 1, 2, 3

# every symbol include/bdfb.h declares
SYMBOLS = ["bdfb_default_options", "bdfb_create", "bdfb_set_model", "bdfb_set_cell_stats", "bdfb_integrate",
           "bdfb_integrate_host", "bdfb_get_stats", "bdfb_last_launch_count", "bdfb_last_kernel_ms",
           "bdfb_destroy", "bdfb_last_error", "bdfb_version", "bdfb_eval_rhs", "bdfb_eval_jac",
           "bdfb_lu_factor_solve", "bdfb_probe_fp64", "bdfb_set_comm", "bdfb_set_kernel", "bdfb_wrms_group",
           "bdfb_phase_ms", "bdfb_minmax", "bdfb_set_atol_typical", "bdfb_set_jacobian",
           "bdfb_split_lu_factor_solve", "bdfb_set_linear_solver", "bdfb_set_method"]


class Options(C.Structure):
    _fields_ = [("qmax", C.c_int32), ("mode", C.c_int32), ("mxstep", C.c_int64), ("h0", C.c_double),
                ("hmin", C.c_double), ("hmax", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("n_cells", C.c_int64), ("n_failed", C.c_int64), ("nst", C.c_int64), ("nfe", C.c_int64),
                ("nje", C.c_int64), ("nsetups", C.c_int64), ("nni", C.c_int64), ("netf", C.c_int64),
                ("ncfn", C.c_int64), ("nst_max", C.c_int64), ("nfe_max", C.c_int64), ("nli", C.c_int64)]


class CellStats(C.Structure):
    _fields_ = [("status", C.c_void_p), ("nst", C.c_void_p), ("nfe", C.c_void_p), ("nje", C.c_void_p),
                ("nsetups", C.c_void_p), ("nni", C.c_void_p), ("netf", C.c_void_p), ("ncfn", C.c_void_p),
                ("q_last", C.c_void_p), ("h_last", C.c_void_p), ("t_reached", C.c_void_p)]


class KwhParams(C.Structure):
    _fields_ = [("z", C.c_double), ("X", C.c_double), ("Y", C.c_double), ("gamma_ad", C.c_double),
                ("gph", C.c_double * 3), ("eph", C.c_double * 3)]


_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load libbdfb.so (fails loudly; no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(f"{LIB_PATH} not built: run __graft_entry__.build() or paper_2405_01713_b200/build.py")
    L = C.CDLL(LIB_PATH)
    vp, dp, i32, i64 = C.c_void_p, C.c_double, C.c_int32, C.c_int64
    L.bdfb_default_options.restype = None
    L.bdfb_default_options.argtypes = [C.POINTER(Options)]
    L.bdfb_create.restype = C.c_int
    L.bdfb_create.argtypes = [C.POINTER(vp), i64, i32, dp, C.POINTER(C.c_double), C.POINTER(Options), i32]
    L.bdfb_set_model.restype = C.c_int
    L.bdfb_set_model.argtypes = [vp, i32, vp, C.c_size_t]
    L.bdfb_set_cell_stats.restype = C.c_int
    L.bdfb_set_cell_stats.argtypes = [vp, C.POINTER(CellStats)]
    L.bdfb_integrate.restype = C.c_int
    L.bdfb_integrate.argtypes = [vp, dp, dp, vp, vp, vp, i32, vp]
    L.bdfb_integrate_host.restype = C.c_int
    L.bdfb_integrate_host.argtypes = [vp, dp, dp, vp, vp, vp, i32, vp]
    L.bdfb_get_stats.restype = i64
    L.bdfb_get_stats.argtypes = [vp, C.POINTER(Stats)]
    L.bdfb_last_launch_count.restype = i32
    L.bdfb_last_launch_count.argtypes = [vp]
    L.bdfb_set_jacobian.restype = C.c_int
    L.bdfb_set_jacobian.argtypes = [vp, i32]
    L.bdfb_set_method.restype = C.c_int
    L.bdfb_set_method.argtypes = [vp, i32]
    L.bdfb_set_linear_solver.restype = C.c_int
    L.bdfb_set_linear_solver.argtypes = [vp, i32, i32]
    L.bdfb_minmax.restype = C.c_int
    L.bdfb_minmax.argtypes = [vp, vp, i32, vp, vp, vp]
    L.bdfb_set_atol_typical.restype = C.c_int
    L.bdfb_set_atol_typical.argtypes = [vp, vp, vp, dp, dp, vp, vp]
    L.bdfb_phase_ms.restype = i32
    L.bdfb_phase_ms.argtypes = [vp, C.POINTER(C.c_double), i32]
    L.bdfb_last_kernel_ms.restype = dp
    L.bdfb_last_kernel_ms.argtypes = [vp]
    L.bdfb_destroy.restype = None
    L.bdfb_destroy.argtypes = [vp]
    L.bdfb_last_error.restype = C.c_char_p
    L.bdfb_last_error.argtypes = [vp]
    L.bdfb_version.restype = C.c_char_p
    L.bdfb_version.argtypes = []
    L.bdfb_eval_rhs.restype = C.c_int
    L.bdfb_eval_rhs.argtypes = [vp, dp, vp, vp, vp, vp, vp, vp]
    L.bdfb_eval_jac.restype = C.c_int
    L.bdfb_eval_jac.argtypes = [vp, dp, vp, vp, vp, vp]
    L.bdfb_lu_factor_solve.restype = C.c_int
    L.bdfb_lu_factor_solve.argtypes = [i32, i64, vp, vp, vp, vp, vp]
    L.bdfb_split_lu_factor_solve.restype = C.c_int
    L.bdfb_split_lu_factor_solve.argtypes = [i32, i64, vp, vp, vp, vp, vp]
    L.bdfb_set_comm.restype = C.c_int
    L.bdfb_set_comm.argtypes = [vp, vp, i32, i32, i64]
    L.bdfb_set_kernel.restype = C.c_int
    L.bdfb_set_kernel.argtypes = [vp, i32]
    L.bdfb_wrms_group.restype = i32
    L.bdfb_wrms_group.argtypes = [vp]
    L.bdfb_probe_fp64.restype = C.c_int
    L.bdfb_probe_fp64.argtypes = [i32, dp, C.POINTER(C.c_double), C.POINTER(C.c_int32)]
    _lib = L
    return L
