"""ctypes binding of include/spotfit.h (libspotfit_b200.so, built in-tree).

There is no CPU fallback: if the library is missing, or a compute entry point
is called without a CUDA device, this module raises.  The CPU restatement in
oracle/ is test infrastructure and is never imported here.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPOTFIT_LIB selects an alternative in-tree build (tools/variants: A/B experiments)
LIB_PATH = os.environ.get("SPOTFIT_LIB") or os.path.join(_HERE, "_lib", "libspotfit_b200.so")

SF_STOP_MAX_ERROR = 0
SF_STOP_MIN_DELTA = 1
SF_STOP_MIN_STEP = 2
SF_STOP_NOT_CONVERGED = 3
SF_STOP_MAX_ITERATIONS = 4
SF_FLAG_INVALID = 0x40
SF_FLAG_NOIMP = 0x80


class sf_config(ctypes.Structure):
    _fields_ = [
        ("model", ctypes.c_int32),
        ("max_iterations", ctypes.c_int32),
        ("max_error", ctypes.c_double),
        ("min_delta", ctypes.c_double),
        ("min_step", ctypes.c_double),
        ("lambda_init", ctypes.c_double),
        ("lambda_up", ctypes.c_double),
        ("lambda_down", ctypes.c_double),
        ("lambda_max", ctypes.c_double),
        ("margin_x", ctypes.c_double),
        ("margin_y", ctypes.c_double),
        ("sigma_min", ctypes.c_double),
        ("sigma_max", ctypes.c_double),
    ]


class sf_stats(ctypes.Structure):
    _fields_ = [
        ("n_gradient_evals", ctypes.c_uint64),
        ("n_trial_evals", ctypes.c_uint64),
        ("n_kernel_evals", ctypes.c_uint64),
        ("h2d_ms", ctypes.c_double),
        ("kernel_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("n_devices", ctypes.c_int32),
        ("n_chunks", ctypes.c_int32),
        ("n_chunks_u16", ctypes.c_int32),
        ("h2d_bytes", ctypes.c_uint64),
    ]


class sf_eval_record(ctypes.Structure):
    _fields_ = [
        ("singular", ctypes.c_int32),
        ("alpha", ctypes.c_float),
        ("beta", ctypes.c_float),
        ("chi", ctypes.c_float),
        ("F", ctypes.c_double),
        ("G", ctypes.c_double),
        ("FF", ctypes.c_double),
        ("FG", ctypes.c_double),
        ("denom", ctypes.c_double),
        ("dF", ctypes.c_double * 4),
        ("dFF", ctypes.c_double * 4),
        ("dFG", ctypes.c_double * 4),
        ("gamma", ctypes.c_double * 4),
        ("dalpha", ctypes.c_double * 4),
        ("dbeta", ctypes.c_double * 4),
        ("rhs", ctypes.c_double * 4),
        ("jtj", ctypes.c_double * 10),
    ]


class sf_sim_config(ctypes.Structure):
    _fields_ = [
        ("model", ctypes.c_int32),
        ("n_signal", ctypes.c_double),
        ("n_background", ctypes.c_double),
        ("sigma_lo", ctypes.c_double),
        ("sigma_hi", ctypes.c_double),
        ("spread", ctypes.c_double),
        ("noise", ctypes.c_int32),
        ("rounding", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
    ]


class sf_csv_col(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("data", ctypes.c_void_p), ("stride", ctypes.c_int64)]


SF_CSV_F32, SF_CSV_U8, SF_CSV_STOP, SF_CSV_FLAGS, SF_CSV_SKIP = range(5)

# symbol -> (restype, argtypes); the exact set include/spotfit.h declares
_vp, _i32, _i64, _f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
SYMBOLS = {
    "sf_fit_batch": (ctypes.c_int, [_vp, _i32, _i32, _i64, _vp, ctypes.POINTER(sf_config), _vp, _vp, _vp, _vp, _vp,
                                    _vp, _vp, _i32, ctypes.POINTER(sf_stats)]),
    "sf_fit_batch_u16": (ctypes.c_int, [_vp, _i32, _i32, _i64, _vp, ctypes.POINTER(sf_config), _vp, _vp, _vp, _vp,
                                        _vp, _vp, _vp, _i32, ctypes.POINTER(sf_stats)]),
    "sf_fit_batch_device": (ctypes.c_int, [_vp, _i32, _i32, _i64, _vp, ctypes.POINTER(sf_config), _vp, _vp, _vp, _vp,
                                           _vp, _vp, _vp, _vp]),
    "sf_fit_batch_device_u16": (ctypes.c_int, [_vp, _i32, _i32, _i64, _vp, ctypes.POINTER(sf_config), _vp, _vp, _vp,
                                               _vp, _vp, _vp, _vp, _vp]),
    "sf_eval_batch_device": (ctypes.c_int, [_vp, _i32, _i32, _i64, _i32, _vp, _vp, _vp]),
    "sf_estimate_initial_device": (ctypes.c_int, [_vp, _i32, _i32, _i64, _i32, _f64, _f64, _vp, _vp, _vp]),
    "sf_model_profile_device": (ctypes.c_int, [_vp, _i32, _i32, _i64, _i32, _vp, _vp, _vp]),
    "sf_model_alpha_beta_device": (ctypes.c_int, [_vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp, _vp]),
    "sf_model_chi_squared_device": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp]),
    "sf_model_gradient_sums_device": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _i64, _vp, _vp]),
    "sf_model_coefficient_gradients_device": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _i64, _vp, _vp, _vp,
                                                             _vp]),
    "sf_model_chi_gradient_device": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i64, _vp, _vp,
                                                    _vp]),
    "sf_simulate_host": (ctypes.c_int, [ctypes.POINTER(sf_sim_config), _i32, _i32, _i64, _i64, _vp, _vp, _i32]),
    "sf_simulate_device": (ctypes.c_int, [ctypes.POINTER(sf_sim_config), _i32, _i32, _i64, _i64, _vp, _vp, _vp]),
    "sf_lane_geometry": (ctypes.c_int, [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sf_debug_npexp_device": (ctypes.c_int, [_vp, _vp, _i64, _i32, _vp]),
    "sf_debug_ddiv_device": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp]),
    "sf_debug_tame_div_device": (ctypes.c_int, [_vp, _vp]),
    "sf_csv_write": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, _i64, _i64, ctypes.c_int,
                                    ctypes.POINTER(sf_csv_col), ctypes.c_int]),
    "sf_csv_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64), _vp, ctypes.c_int,
                                   ctypes.POINTER(sf_csv_col), _i64, ctypes.c_int]),
    "sf_format_f32": (ctypes.c_int, [_vp, _i64, _vp, _i64, ctypes.POINTER(ctypes.c_int64)]),
    "sf_csv_last_error": (ctypes.c_char_p, []),
    "sf_shard_range": (ctypes.c_int, [_i64, _i32, _i32, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "sf_debug_narrow_u16": (ctypes.c_int, [_vp, _i64, _vp, _i32]),
    "sf_debug_par_copy": (ctypes.c_int, [_vp, _vp, _i64, _i32]),
    "sf_host_alloc": (ctypes.c_void_p, [ctypes.c_size_t]),
    "sf_host_free": (None, [_vp]),
    "sf_device_count": (ctypes.c_int, []),
    "sf_last_error": (ctypes.c_char_p, []),
    "sf_version": (ctypes.c_int, []),
}

_lib = None
_lock = threading.Lock()


class SpotfitError(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise SpotfitError(
                        f"{LIB_PATH} is missing: build it with `python -m paper_2106_02045_b200.build` "
                        "(there is no CPU fallback)")
                L = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SYMBOLS.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise SpotfitError(lib().sf_last_error().decode(errors="replace"))


def require_gpu() -> None:
    if lib().sf_device_count() < 1:
        raise SpotfitError("no CUDA device visible: the spotfit B200 engine has no CPU fallback")
