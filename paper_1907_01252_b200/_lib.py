"""ctypes binding of the C ABI in include/pint_b200.h.

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is no fallback: importing the product path without the
library raises, so a missing extension can never silently route through a CPU
implementation.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PINT_LIB") or os.path.join(_HERE, "libpint_b200.so")

PINT_OK = 0
PINT_NUMERIC_BREAKDOWN = 1
PINT_NEWTON_MAX_ITERS = 2
PINT_MESH_DEGENERATE = 3
PINT_INVALID_ARG = 4
PINT_CUDA_ERROR = 5

STATUS_NAMES = {
    PINT_OK: "ok",
    PINT_NUMERIC_BREAKDOWN: "numeric breakdown",
    PINT_NEWTON_MAX_ITERS: "Newton iteration budget exhausted",
    PINT_MESH_DEGENERATE: "degenerate mesh",
    PINT_INVALID_ARG: "invalid argument",
    PINT_CUDA_ERROR: "CUDA error",
}

# every symbol include/pint_b200.h declares (tests check the export table)
EXPORTS = (
    "pint_create", "pint_create_ex", "pint_destroy", "pint_last_error", "pint_sizes", "pint_level0_fp32", "pint_flags",
    "pint_propagate", "pint_residual", "pint_jvp", "pint_assemble", "pint_jacobian_blocks",
    "pint_spmv", "pint_precond_setup", "pint_precond_apply", "pint_linear_solve",
    "pint_parareal_precorrect", "pint_parareal_correct_one", "pint_profile", "pint_profile_read",
    "pint_profile_kernel", "pint_coarse_sweep", "pint_boundary_error", "pint_linear_solve_mf",
)

PINT_CTX_MATRIX_FREE = 1


class ProblemDesc(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int32),
        ("cells", ctypes.c_int32 * 3),
        ("extent", ctypes.c_double * 3),
        ("bar_lo", ctypes.c_double * 3),
        ("bar_hi", ctypes.c_double * 3),
        ("rho_f", ctypes.c_double),
        ("nu_f", ctypes.c_double),
        ("rho_s", ctypes.c_double),
        ("mu_s", ctypes.c_double),
        ("lambda_s", ctypes.c_double),
        ("u_peak", ctypes.c_double),
        ("ramp_time", ctypes.c_double),
        ("alpha_p", ctypes.c_double),
        ("stab_k", ctypes.c_double),
    ]


class NewtonOpts(ctypes.Structure):
    _fields_ = [
        ("abs_tol", ctypes.c_double),
        ("rel_tol", ctypes.c_double),
        ("max_iters", ctypes.c_int32),
        ("damping_min", ctypes.c_double),
    ]


class KrylovOpts(ctypes.Structure):
    _fields_ = [
        ("rtol", ctypes.c_double),
        ("atol", ctypes.c_double),
        ("restart", ctypes.c_int32),
        ("max_iters", ctypes.c_int32),
        ("pre_smooth", ctypes.c_int32),
        ("post_smooth", ctypes.c_int32),
        ("omega", ctypes.c_double),
        ("max_levels", ctypes.c_int32),
        ("coarse_sweeps", ctypes.c_int32),
        ("smoother", ctypes.c_int32),
        ("precond_reuse", ctypes.c_int32),
        ("rtol_first", ctypes.c_double),
    ]


_P = ctypes.c_void_p
_I = ctypes.c_int32
_D = ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)
_IP = ctypes.POINTER(ctypes.c_int32)

_SIGNATURES = {
    "pint_create": (_I, [ctypes.POINTER(ProblemDesc), _I, _I, ctypes.POINTER(_P)]),
    "pint_create_ex": (_I, [ctypes.POINTER(ProblemDesc), _I, _I, _I, ctypes.POINTER(_P)]),
    "pint_linear_solve_mf": (_I, [_P, _I, _P, _P, _DP, _DP, _DP, _P, _P, ctypes.POINTER(KrylovOpts), _IP, _DP,
                                  _P]),
    "pint_destroy": (_I, [_P]),
    "pint_last_error": (ctypes.c_char_p, [_P]),
    "pint_sizes": (_I, [_P, _IP, _IP, _IP, _IP]),
    "pint_level0_fp32": (_I, [_P, _IP]),
    "pint_flags": (_I, [_P, ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(ctypes.c_uint8)]),
    "pint_propagate": (_I, [_P, _I, _P, _P, _DP, _DP, _IP, _D, _D, ctypes.POINTER(NewtonOpts),
                            ctypes.POINTER(KrylovOpts), _IP, _IP, _IP, _DP, _P]),
    "pint_residual": (_I, [_P, _I, _P, _P, _DP, _DP, _DP, _P, _DP, _P]),
    "pint_jvp": (_I, [_P, _I, _P, _P, _P, _DP, _DP, _DP, _P, _P]),
    "pint_assemble": (_I, [_P, _I, _P, _P, _DP, _DP, _DP, _P]),
    "pint_jacobian_blocks": (_I, [_P, _I, _P, _P]),
    "pint_spmv": (_I, [_P, _I, _P, _P, _P]),
    "pint_precond_setup": (_I, [_P, _I, ctypes.POINTER(KrylovOpts), _P]),
    "pint_precond_apply": (_I, [_P, _I, _P, _P, _P]),
    "pint_linear_solve": (_I, [_P, _I, _P, _P, ctypes.POINTER(KrylovOpts), _IP, _DP, _P]),
    "pint_parareal_precorrect": (_I, [_I, _I, _I, _I, _P, _P, _P, _P]),
    "pint_parareal_correct_one": (_I, [_I, _I, _I, _P, _P, _P, _P, _P, _I, _D, _D, _DP, _DP, _P]),
    "pint_coarse_sweep": (_I, [_P, _I, _P, _P, _P, _P, _P, _DP, _IP, _D, _D, ctypes.POINTER(NewtonOpts),
                               ctypes.POINTER(KrylovOpts), _I, _D, _D, _DP, _DP, _IP, _IP, _IP, _DP, _P]),
    "pint_boundary_error": (_I, [_P, _I, _P, _P, _DP, _IP, _P]),
    "pint_profile": (_I, [_P, _I]),
    "pint_profile_kernel": (ctypes.c_char_p, [_P]),
    "pint_profile_read": (_I, [_P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                               ctypes.POINTER(ctypes.c_int64), _DP, ctypes.POINTER(ctypes.c_int64)]),
}

_lib = None


class LibraryMissing(ImportError):
    pass


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the shared library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryMissing(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols(path: str = LIB_PATH):
    """Names from EXPORTS that the library actually exports (no GPU needed)."""
    lib = ctypes.CDLL(path)
    out = []
    for name in EXPORTS:
        try:
            getattr(lib, name)
            out.append(name)
        except AttributeError:
            pass
    return out
