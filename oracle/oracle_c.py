"""ctypes front end of the C restatement (oracle/spotfit_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  Never by the product.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libspotfit_oracle.so")


def build(force: bool = False) -> str:
    src = [os.path.join(_HERE, f) for f in ("spotfit_oracle.c", "spotfit_oracle.h", "Makefile")]
    if force or not os.path.exists(_SO) or any(os.path.getmtime(s) > os.path.getmtime(_SO) for s in src):
        subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    return _SO


class OracleConfig(ctypes.Structure):
    _fields_ = [
        ("max_iterations", ctypes.c_int),
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


class OracleEval(ctypes.Structure):
    _fields_ = [
        ("singular", ctypes.c_int),
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
        ("rhs", ctypes.c_double * 5),
        ("jtj", ctypes.c_double * 15),
    ]


EVAL_DTYPE = np.dtype(
    [
        ("singular", np.int32),
        ("alpha", np.float32),
        ("beta", np.float32),
        ("chi", np.float32),
        ("F", np.float64),
        ("G", np.float64),
        ("FF", np.float64),
        ("FG", np.float64),
        ("denom", np.float64),
        ("dF", np.float64, 4),
        ("dFF", np.float64, 4),
        ("dFG", np.float64, 4),
        ("gamma", np.float64, 4),
        ("dalpha", np.float64, 4),
        ("dbeta", np.float64, 4),
        ("rhs", np.float64, 5),
        ("jtj", np.float64, 15),
    ],
    align=True,
)

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        f32p = np.ctypeslib.ndpointer(np.float32, flags="C")
        u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
        _lib.npexp_f32.restype = ctypes.c_float
        _lib.npexp_f32.argtypes = [ctypes.c_float]
        _lib.npexp_f32_array.argtypes = [f32p, f32p, ctypes.c_int64]
        _lib.npexp_f32_clamped.restype = ctypes.c_float
        _lib.npexp_f32_clamped.argtypes = [ctypes.c_float]
        _lib.npexp_clamp_mismatches.restype = ctypes.c_int64
        _lib.npexp_clamp_mismatches.argtypes = [ctypes.c_float, ctypes.c_float]
        _lib.pw_sum.restype = ctypes.c_double
        _lib.pw_sum.argtypes = [f32p, ctypes.c_int]
        _lib.sf_oracle_solve.restype = ctypes.c_int
        _lib.sf_oracle_solve.argtypes = [
            ctypes.c_int,
            np.ctypeslib.ndpointer(np.float64, flags="C"),
            np.ctypeslib.ndpointer(np.float64, flags="C"),
            ctypes.c_double,
            np.ctypeslib.ndpointer(np.float64, flags="C"),
        ]
        _lib.sf_oracle_fit_batch.restype = ctypes.c_int
        _lib.sf_oracle_fit_batch.argtypes = [
            f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int, f32p,
            ctypes.POINTER(OracleConfig), f32p, f32p, f32p, f32p, u8p, u8p, ctypes.c_int,
        ]
        _lib.sf_oracle_eval_batch.restype = ctypes.c_int
        _lib.sf_oracle_eval_batch.argtypes = [
            f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int, f32p, ctypes.c_void_p, ctypes.c_int,
        ]
        _lib.sf_oracle_eval_size.restype = ctypes.c_int
        assert _lib.sf_oracle_eval_size() == EVAL_DTYPE.itemsize, "EVAL_DTYPE layout mismatch"
    return _lib


def npexp(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty_like(x)
    lib().npexp_f32_array(x.ravel(), y.ravel(), x.size)
    return y


def pw_sum(x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    return lib().pw_sum(x, x.size)


def solve(jtj_packed, rhs, lam):
    P = len(rhs)
    d = np.zeros(P, np.float64)
    ok = lib().sf_oracle_solve(P, np.ascontiguousarray(jtj_packed, np.float64), np.ascontiguousarray(rhs, np.float64),
                               float(lam), d)
    return bool(ok), d


def make_config(cfg) -> OracleConfig:
    """cfg: any object with the FitConfig field names (paper defaults)."""
    return OracleConfig(
        int(cfg.max_iterations), float(cfg.max_error), float(cfg.min_delta), float(cfg.min_step),
        float(cfg.lambda_init), float(cfg.lambda_up), float(cfg.lambda_down), float(cfg.lambda_max),
        float(cfg.margin_x), float(cfg.margin_y), float(cfg.sigma_min), float(cfg.sigma_max),
    )


def eval_batch(images: np.ndarray, params: np.ndarray, W: int, H: int, threads: int = 0) -> np.ndarray:
    images = np.ascontiguousarray(images, np.float32)
    params = np.ascontiguousarray(params, np.float32)
    count, P = params.shape
    out = np.zeros(count, EVAL_DTYPE)
    rc = lib().sf_oracle_eval_batch(images.ravel(), W, H, count, P, params.ravel(), out.ctypes.data,
                                    threads or os.cpu_count())
    if rc != 0:
        raise ValueError("oracle eval failed")
    return out


def fit_batch(images: np.ndarray, inits: np.ndarray, W: int, H: int, cfg, threads: int = 0) -> dict:
    images = np.ascontiguousarray(images, np.float32)
    inits = np.ascontiguousarray(inits, np.float32)
    count, P = inits.shape
    out = {
        "params": np.zeros((count, P), np.float32),
        "alpha": np.zeros(count, np.float32),
        "beta": np.zeros(count, np.float32),
        "nchi2": np.zeros(count, np.float32),
        "status": np.zeros(count, np.uint8),
        "iterations": np.zeros(count, np.uint8),
    }
    c = make_config(cfg)
    rc = lib().sf_oracle_fit_batch(
        images.ravel(), W, H, count, P, inits.ravel(), ctypes.byref(c), out["params"].ravel(), out["alpha"],
        out["beta"], out["nchi2"], out["status"], out["iterations"], threads or os.cpu_count(),
    )
    if rc != 0:
        raise ValueError("oracle fit failed")
    return out
