"""ctypes binding of libsptb.so (the C ABI declared in include/sptb.h).

There is deliberately no fallback: if the shared library is missing the
import fails loudly and tells the caller how to build it.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPTB_LIB_VARIANT: an alternative in-tree build (kernel tuning experiments)
LIB_PATH = os.path.join(_HERE, os.environ.get("SPTB_LIB_VARIANT", "libsptb.so"))

OK, ERR_SHAPE, ERR_ARG, ERR_NEAR_ZERO, ERR_CUDA, ERR_CUFFT, ERR_OOM, ERR_NONFINITE, \
    ERR_DIVERGENCE, ERR_STATE = range(10)
PREC_F32, PREC_F64 = 0, 1
FMT_F32, FMT_F64, FMT_REAL, FMT_COMPLEX = 0x0, 0x1, 0x0, 0x2
MAT_S, MAT_SH, MAT_SW = 0, 1, 2
KERNEL_KB, KERNEL_GAUSS = 0, 1
ALGO = {"fbp": 0, "sirt": 1, "cgls": 2, "tv": 3}


class Geometry(C.Structure):
    _fields_ = [("n_p", C.c_int32), ("n_theta", C.c_int32), ("n_x", C.c_int32),
                ("n_y", C.c_int32), ("center", C.c_double),
                ("cos_theta", C.POINTER(C.c_double)), ("sin_theta", C.POINTER(C.c_double))]


class Kernel(C.Structure):
    _fields_ = [("family", C.c_int32), ("width", C.c_int32), ("beta", C.c_double),
                ("sigma", C.c_double)]


class SolverConfig(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("max_iter", C.c_int32), ("tol", C.c_double),
                ("mu", C.c_double), ("tv_inner_iter", C.c_int32), ("bb_enabled", C.c_int32),
                ("nonneg", C.c_int32), ("cgs_mode", C.c_int32)]


# (name, restype, argtypes) for every entry point in include/sptb.h
_P = C.c_void_p
SIGNATURES = [
    ("sptb_last_error", C.c_char_p, []),
    ("sptb_version", C.c_int32, []),
    ("sptb_launch_count", C.c_int64, []),
    ("sptb_fft_count", C.c_int64, []),
    ("sptb_time_spmm", C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                 C.POINTER(C.c_int64)]),
    ("sptb_plan_create", C.c_int, [C.POINTER(_P), C.POINTER(Geometry), C.POINTER(Kernel),
                                   C.c_int32, C.c_int32, C.c_int32, C.c_double]),
    ("sptb_plan_destroy", C.c_int, [_P]),
    ("sptb_reload_switches", C.c_int, []),
    ("sptb_plan_set_stream", C.c_int, [_P, _P]),
    ("sptb_plan_set_filter", C.c_int, [_P, C.POINTER(C.c_double), C.c_int64]),
    ("sptb_plan_calibrate", C.c_int, [_P, C.POINTER(C.c_double)]),
    ("sptb_density_filter", C.c_int, [_P, C.c_int32, C.c_double, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
    ("sptb_plan_set_calibration", C.c_int, [_P, C.c_double]),
    ("sptb_plan_matrix_info", C.c_int, [_P, C.c_int32, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("sptb_plan_matrix_copy", C.c_int, [_P, C.c_int32, _P, _P, _P]),
    ("sptb_plan_deapo_copy", C.c_int, [_P, _P]),
    ("sptb_radon", C.c_int, [_P, _P, C.c_int32, _P, C.c_int32, C.c_int64]),
    ("sptb_radon_adjoint", C.c_int, [_P, _P, C.c_int32, _P, C.c_int32, C.c_int64]),
    ("sptb_iradon", C.c_int, [_P, _P, C.c_int32, _P, C.c_int32, C.c_int64]),
    ("sptb_apply_weights", C.c_int, [_P, _P, C.c_int32, _P, C.c_int32, C.c_int64]),
    ("sptb_backproject", C.c_int, [_P, C.c_int32, C.c_double, _P, C.c_int32, _P, C.c_int32,
                                   C.c_int64]),
    ("sptb_spectral_apply", C.c_int, [_P, C.POINTER(C.c_double), C.c_int64, _P, C.c_int32, _P,
                                      C.c_int32, C.c_int64]),
    ("sptb_spmm", C.c_int, [_P, C.c_int32, _P, _P, C.c_int64, C.c_int32]),
    ("sptb_solve", C.c_int, [_P, C.POINTER(SolverConfig), _P, C.c_int32, _P, C.c_int32,
                             C.c_int64, _P, _P, _P, _P]),
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the B200 kernels are not built. Run "
            "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a). "
            "There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

_EXC = {
    ERR_SHAPE: errors.ShapeMismatchError,
    ERR_ARG: ValueError,
    ERR_NEAR_ZERO: errors.NearZeroDenominatorError,
    ERR_CUDA: RuntimeError,
    ERR_CUFFT: RuntimeError,
    ERR_OOM: MemoryError,
    ERR_NONFINITE: errors.NonFiniteError,
    ERR_DIVERGENCE: errors.DivergenceError,
    ERR_STATE: RuntimeError,
}


def last_error() -> str:
    msg = lib.sptb_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map a status code to the reference's exception types."""
    if rc == OK:
        return
    exc = _EXC.get(rc, RuntimeError)
    raise exc(f"{what}: {last_error()}" if what else last_error())


def launch_count() -> int:
    return int(lib.sptb_launch_count())
