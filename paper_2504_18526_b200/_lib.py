"""ctypes binding of libsisdc_b200.so (include/sisdc_b200.h).

The product path has no CPU fallback: if the library (built in-tree by
``paper_2504_18526_b200/build.py``) or a CUDA device is missing, every entry
point raises.  Device buffers are torch float64 CUDA tensors used purely as
allocations; all arithmetic happens in the library's sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SISDC_LIB", os.path.join(HERE, "libsisdc_b200.so"))   # override: A/B experiments

OK, ERR_ARG, ERR_CUDA, ERR_NONFINITE, ERR_NOCONV, ERR_UNSUPPORTED = range(6)
CONVDIFF, BURGERS, EULER2D, ADVECTION2D, BURGERS2D, CNS1D, NS2D = 0, 1, 2, 3, 4, 5, 6
PERIODIC, DIRICHLET = 0, 1
SCHEMES = {"euler": 0, "si1": 1, "si2": 2}
COEF_NONE, COEF_CONST, COEF_FIELD, COEF_SI, COEF_PHYS, COEF_MATRIX = range(6)


class SolverError(RuntimeError):
    """Raised when the discrete solver breaks down (``dgsem.py:29-30``)."""


class LibraryError(RuntimeError):
    """CUDA / ABI failure of the native library."""


class Coef(C.Structure):
    _fields_ = [("kind", C.c_int), ("value", C.c_double), ("ptr", C.c_void_p)]


class Op2DDesc(C.Structure):
    _fields_ = [("nex", C.c_int), ("ney", C.c_int), ("degree", C.c_int), ("ncomp", C.c_int), ("problem", C.c_int),
                ("x_left", C.c_double), ("x_right", C.c_double), ("y_bottom", C.c_double), ("y_top", C.c_double),
                ("gamma", C.c_double), ("nu", C.c_double), ("ax", C.c_double), ("ay", C.c_double),
                ("penalty", C.c_double), ("prandtl", C.c_double)]


class Op1DDesc(C.Structure):
    _fields_ = [("n_elem", C.c_int), ("degree", C.c_int), ("ncomp", C.c_int), ("bc", C.c_int),
                ("problem", C.c_int), ("x_left", C.c_double), ("x_right", C.c_double),
                ("speed", C.c_double), ("nu", C.c_double), ("penalty", C.c_double),
                ("gamma", C.c_double), ("eta", C.c_double), ("prandtl", C.c_double)]


P = C.c_void_p
D = C.c_double
I = C.c_int
DP = C.POINTER(C.c_double)

# name -> (restype, argtypes); the authoritative list of exports (tests check
# that every symbol declared in include/sisdc_b200.h is bound here).
SIGNATURES = {
    "sisdc_abi_version": (I, []),
    "sisdc_struct_size": (I, [I]),
    "sisdc_ctx_create": (I, [I, C.POINTER(P)]),
    "sisdc_ctx_destroy": (None, [P]),
    "sisdc_ctx_last_error": (C.c_char_p, [P]),
    "sisdc_ctx_set_stream": (I, [P, P]),
    "sisdc_ctx_synchronize": (I, [P]),
    "sisdc_ctx_set_cg": (I, [P, D, I, I]),
    "sisdc_ctx_status": (I, [P, C.POINTER(I), C.POINTER(I), C.POINTER(I)]),
    "sisdc_ctx_reset_status": (I, [P]),
    "sisdc_ctx_reset_log": (I, [P]),
    "sisdc_ctx_cg_log": (I, [P, I, C.POINTER(I), DP, C.POINTER(I)]),
    "sisdc_ctx_launch_count": (C.c_int64, [P]),
    "sisdc_ctx_debug_timing": (I, [P, C.POINTER(C.c_longlong), I]),
    "sisdc_copy": (I, [P, P, P, C.c_int64]),
    "sisdc_lincomb": (I, [P, C.c_int64, DP, P, P, P, P, P]),
    "sisdc_op1d_create": (I, [P, C.POINTER(Op1DDesc), C.POINTER(P)]),
    "sisdc_op2d_create": (I, [P, C.POINTER(Op2DDesc), C.POINTER(P)]),
    "sisdc_op1d_destroy": (None, [P]),
    "sisdc_op1d_tables": (I, [P, DP, DP, DP]),
    "sisdc_op1d_set_nu_art": (I, [P, P]),
    "sisdc_op1d_set_boundary": (I, [P, I, DP, DP, DP]),
    "sisdc_smooth_start": (I, [P, I, P, P]),
    "sisdc_persson_viscosity": (I, [P, P, D, D, P]),
    "sisdc_apply_convection": (I, [P, P, D, P]),
    "sisdc_apply_diffusion": (I, [P, Coef, P, D, P]),
    "sisdc_eval_rhs": (I, [P, P, D, P]),
    "sisdc_coef_field": (I, [P, Coef, P]),
    "sisdc_implicit_solve": (I, [P, Coef, D, P, D, P]),
    "sisdc_stage_rhs": (I, [P, P, P, D, P, I, DP, D, P, P, D, P, P]),
    "sisdc_stage_solve": (I, [P, Coef, D, P, P, D, P, I, DP, D, P, P, D, D, P, P, P]),
    "sisdc_node_caches": (I, [P, I, I, I, I, P, P, P, DP, D, DP, P, P, P]),
    "sisdc_eval_rhs_nodes": (I, [P, I, P, DP, P]),
    "sisdc_collocation_defect": (I, [P, I, DP, D, I, P, P, P, D, P, P]),
    "sisdc_xfer_create": (I, [P, I, I, I, I, I, DP, DP, DP, DP, DP, C.POINTER(P)]),
    "sisdc_xfer2d_create": (I, [P, I, I, I, I, I, DP, DP, DP, DP, DP, C.POINTER(P)]),
    "sisdc_xfer_destroy": (None, [P]),
    "sisdc_xfer_spatial": (I, [P, I, P, P]),
    "sisdc_xfer_down": (I, [P, I, I, P, P]),
    "sisdc_xfer_fas_restrict": (I, [P, DP, D, I, P, P, P, P, P, P]),
    "sisdc_xfer_interp": (I, [P, I, P, P, P]),
    "sisdc_nccl_unique_id": (I, [C.c_char_p]),
    "sisdc_comm_create": (I, [P, C.c_char_p, I, I, C.POINTER(P)]),
    "sisdc_comm_destroy": (None, [P]),
    "sisdc_op2d_create_part": (I, [P, C.POINTER(Op2DDesc), I, I, I, P, C.POINTER(P)]),
    "sisdc_op2d_part_layout": (I, [P, I, C.POINTER(I), C.POINTER(I), C.POINTER(C.c_int64), C.POINTER(I)]),
    "sisdc_halo_exchange": (I, [P, P, I, C.c_int64, I]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and bind the native library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryError(
            f"{path} is missing: build it with `python -m paper_2504_18526_b200.build` "
            "(there is no CPU fallback for the sweep path)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.sisdc_abi_version() != 2:
        raise LibraryError("ABI version mismatch")
    for which, st in enumerate((Op1DDesc, Op2DDesc, Coef)):
        if lib.sisdc_struct_size(which) != C.sizeof(st):
            raise LibraryError(f"ABI struct {st.__name__} is {C.sizeof(st)} bytes here, "
                               f"{lib.sisdc_struct_size(which)} in the library")
    _lib = lib
    return lib


def darr(a) -> "C.Array":
    """Host float64 array -> ctypes double pointer (kept alive by caller)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(DP)


def ptr(t) -> int | None:
    """Device pointer of a torch CUDA float64 tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()
