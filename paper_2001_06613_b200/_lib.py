"""ctypes binding of the C-ABI engine (include/seqreg_b200.h).

This is the only place the shared library is loaded.  There is no CPU fallback:
if ``libseqreg_b200.so`` is missing or no CUDA device is present, the product
path raises (``EngineUnavailable``).  Tests that only check the ABI surface use
:func:`load_library` without creating a context.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

__all__ = [
    "EngineUnavailable",
    "SR_OK",
    "SR_ERR_ARG",
    "SR_ERR_CUDA",
    "SR_ERR_SINGULAR",
    "SR_ERR_UNSUPPORTED",
    "SR_ERR_CALLBACK",
    "SrLbfgsOptions",
    "SrLbfgsResult",
    "OBJECTIVE_FN",
    "TRACE_FN",
    "SR_F32",
    "SR_F64",
    "SR_NCC",
    "SR_NGF",
    "SR_AFFINE",
    "SR_DISPLACEMENT",
    "SR_MAX_FRAMES",
    "SrGrid",
    "SrProblem",
    "EXPORTS",
    "library_path",
    "load_library",
    "check",
]

SR_OK, SR_ERR_ARG, SR_ERR_CUDA, SR_ERR_SINGULAR, SR_ERR_UNSUPPORTED, SR_ERR_CALLBACK = 0, 1, 2, 3, 4, 5
SR_F32, SR_F64 = 0, 1
SR_NCC, SR_NGF = 0, 1
SR_AFFINE, SR_DISPLACEMENT = 0, 1
SR_MAX_FRAMES = 160

_LIBNAME = "libseqreg_b200.so"


class EngineUnavailable(RuntimeError):
    """The CUDA engine cannot run here (library not built, or no GPU)."""


class SrGrid(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int32),
        ("dims", ctypes.c_int32 * 3),
        ("spacing", ctypes.c_double * 3),
        ("origin", ctypes.c_double * 3),
    ]


class SrProblem(ctypes.Structure):
    _fields_ = [
        ("grid", SrGrid),
        ("dtype", ctypes.c_int32),
        ("feature", ctypes.c_int32),
        ("param", ctypes.c_int32),
        ("ngf_eps", ctypes.c_double),
        ("k", ctypes.c_int32),
        ("frame_index", ctypes.POINTER(ctypes.c_int32)),
        ("frames_dev", ctypes.c_void_p),
        ("nframes", ctypes.c_int32),
        ("shifts_dev", ctypes.c_void_p),
        ("pix_lo", ctypes.c_int64),
        ("pix_hi", ctypes.c_int64),
        ("y_dev", ctypes.c_void_p),
        ("y_off", ctypes.c_int64),
        ("y_stride", ctypes.c_int64),
        ("affine", ctypes.POINTER(ctypes.c_double)),
    ]


class SrLbfgsOptions(ctypes.Structure):
    _fields_ = [
        ("memory", ctypes.c_int32),
        ("max_iters", ctypes.c_int32),
        ("grad_tol", ctypes.c_double),
        ("step_tol", ctypes.c_double),
        ("f_tol", ctypes.c_double),
        ("armijo_c1", ctypes.c_double),
        ("backtrack_factor", ctypes.c_double),
        ("max_backtracks", ctypes.c_int32),
    ]


class SrLbfgsResult(ctypes.Structure):
    _fields_ = [
        ("f_final", ctypes.c_double),
        ("f_initial", ctypes.c_double),
        ("iterations", ctypes.c_int32),
        ("objective_evaluations", ctypes.c_int32),
        ("converged_reason", ctypes.c_int32),
    ]


# objective(user, x_dev, f_out, g_dev) -> status; trace(user, iteration, f, grad_inf, step, evaluations)
OBJECTIVE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                ctypes.c_void_p)
TRACE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int32, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                            ctypes.c_int32)

_c = ctypes
_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_I32P = ctypes.POINTER(ctypes.c_int32)
_U8P = ctypes.POINTER(ctypes.c_uint8)
_PROB = ctypes.POINTER(SrProblem)

# name -> (restype, argtypes); exactly the declarations of include/seqreg_b200.h
EXPORTS = {
    "sr_raw_size": (_c.c_int64, [_c.c_int32]),
    "sr_stats_size": (_c.c_int64, [_c.c_int32]),
    "sr_stats_offset": (_c.c_int64, [_c.c_int32, _c.c_int32]),
    "sr_abi_version": (_c.c_int, []),
    "sr_last_error": (_c.c_char_p, []),
    "sr_status_string": (_c.c_char_p, [_c.c_int]),
    "sr_create": (_c.c_int, [_c.c_int32, _c.POINTER(_P)]),
    "sr_destroy": (_c.c_int, [_P]),
    "sr_set_stream": (_c.c_int, [_P, _P]),
    "sr_set_grid_ctas": (_c.c_int, [_P, _c.c_int32]),
    "sr_set_sample_reuse": (_c.c_int, [_P, _c.c_int32]),
    "sr_frame_shifts": (_c.c_int, [_P, _c.c_int32, _P, _c.c_int32, _c.c_int64, _P]),
    "sr_corr_partial": (_c.c_int, [_P, _PROB, _P]),
    "sr_corr_finalize": (_c.c_int, [_P, _PROB, _P, _D, _c.c_double, _c.c_int64, _P]),
    "sr_grad": (_c.c_int, [_P, _PROB, _P, _P, _c.c_int64, _c.c_int64]),
    "sr_evaluate": (_c.c_int, [_P, _PROB, _D, _c.c_double, _P, _P, _P]),
    "sr_evaluate_reg": (_c.c_int, [_P, _PROB, _D, _c.c_double, _c.c_double, _P, _P, _P, _P]),
    "sr_sample": (_c.c_int, [_P, _PROB, _P]),
    "sr_curvature": (
        _c.c_int,
        [_P, _PROB, _c.c_double, _c.c_double, _P, _c.c_int64, _c.c_int64, _P],
    ),
    "sr_ls_predict": (
        _c.c_int,
        [_P, _c.c_int32, _c.c_int32, _c.c_int64, _U8P, _c.c_double, _P, _P, _P],
    ),
    "sr_interp_linear": (
        _c.c_int,
        [_P, _c.c_int32, _c.c_int32, _c.c_int64, _I32P, _I32P, _D, _P, _P],
    ),
    "sr_pyramid_step": (_c.c_int, [_P, _c.c_int32, _c.c_int32, _I32P, _c.c_int32, _P, _P]),
    "sr_prolong_field": (_c.c_int, [_P, _c.c_int32, _c.POINTER(SrGrid), _c.POINTER(SrGrid), _c.c_int32, _P, _P]),
    "sr_lbfgs_defaults": (None, [_c.POINTER(SrLbfgsOptions)]),
    "sr_lbfgs_minimize": (
        _c.c_int,
        [_P, _c.c_int64, _P, _c.POINTER(SrLbfgsOptions), OBJECTIVE_FN, _P, TRACE_FN, _P, _c.POINTER(SrLbfgsResult)],
    ),
}

_lib = None


def library_path() -> Path:
    env = os.environ.get("SEQREG_B200_LIB")
    if env:
        return Path(env)
    return Path(__file__).resolve().parent / _LIBNAME


def load_library():
    """Load the shared library and declare every export (no CUDA call is made)."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not path.exists():
        raise EngineUnavailable(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.sr_abi_version() != 1:
        raise EngineUnavailable("ABI version mismatch")
    _lib = lib
    return lib


class SeqregDeviceError(RuntimeError):
    pass


class SingularSystemError(ValueError):
    """Mirror of seqreg.temporal.SingularSystemError (temporal.py:141-142)."""


def check(status: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if status == SR_OK:
        return
    msg = _lib.sr_last_error().decode(errors="replace") if _lib is not None else ""
    if status == SR_ERR_ARG:
        raise ValueError(msg)
    if status == SR_ERR_SINGULAR:
        raise SingularSystemError(msg)
    if status == SR_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise SeqregDeviceError(msg)
