"""LM solver front end: FitConfig, ParameterBounds, StopReason, FitResult,
fit_single.  Mirrors the reference's lm_solver module; the
state machine itself (pinned in DESIGN.md 3) runs inside
the CUDA kernel (csrc/sf_fit_kernel.cuh:lm_step).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .model import Amplitudes, EllipticalParams, PixelGrid, ShapeParams, SpotImage


class StopReason(enum.IntEnum):
    """SPEC.md:183-186; values equal the low 3 bits of the status byte."""

    MaxError = _lib.SF_STOP_MAX_ERROR
    MinDelta = _lib.SF_STOP_MIN_DELTA
    MinStep = _lib.SF_STOP_MIN_STEP
    NotConverged = _lib.SF_STOP_NOT_CONVERGED
    MaxIterations = _lib.SF_STOP_MAX_ITERATIONS


@dataclass(frozen=True)
class ParameterBounds:
    """SPEC.md:168-171; defaults SPEC.md:248 (margin S/2, sigma in [0.3, S])."""

    margin_x: float
    margin_y: float
    sigma_min: float = 0.3
    sigma_max: float = 0.0

    def __post_init__(self):
        if not self.sigma_min > 0 or not self.sigma_max > self.sigma_min:
            raise ValueError("need 0 < sigma_min < sigma_max")
        if self.margin_x < 0 or self.margin_y < 0:
            raise ValueError("margins must be >= 0")

    @staticmethod
    def for_grid(grid: PixelGrid) -> "ParameterBounds":
        return ParameterBounds(grid.width / 2, grid.height / 2, 0.3, float(max(grid.width, grid.height)))


@dataclass(frozen=True)
class FitConfig:
    """SPEC.md:163-166 with the paper's defaults."""

    max_iterations: int = 20
    max_error: float = 0.0
    min_delta: float = 1e-6
    min_step: float = 1e-4
    lambda_init: float = 0.01
    lambda_up: float = 10.0
    lambda_down: float = 10.0
    lambda_max: float = 1e4
    bounds: Optional[ParameterBounds] = None

    def __post_init__(self):
        if not 1 <= self.max_iterations <= 255:
            raise ValueError("max_iterations must be in [1, 255]")
        if not (self.min_delta > 0 and self.min_step > 0 and self.max_error >= 0):
            raise ValueError("thresholds must be > 0 (max_error >= 0)")
        if not 0 < self.lambda_init < self.lambda_max:
            raise ValueError("need 0 < lambda_init < lambda_max")
        if not (self.lambda_up > 1 and self.lambda_down > 1):
            raise ValueError("lambda factors must be > 1")

    def resolved_bounds(self, grid: PixelGrid) -> ParameterBounds:
        return self.bounds if self.bounds is not None else ParameterBounds.for_grid(grid)

    def to_c(self, grid: PixelGrid, model: int) -> _lib.sf_config:
        b = self.resolved_bounds(grid)
        return _lib.sf_config(model, self.max_iterations, self.max_error, self.min_delta, self.min_step,
                              self.lambda_init, self.lambda_up, self.lambda_down, self.lambda_max, b.margin_x,
                              b.margin_y, b.sigma_min, b.sigma_max)


@dataclass(frozen=True)
class FitResult:
    """SPEC.md:178-181 (+ the no-improvement and invalid-input flags)."""

    shape: object  # ShapeParams or EllipticalParams
    amps: Amplitudes
    stop: StopReason
    iterations_used: int
    normalized_chi2: float
    no_improvement: bool = False
    invalid_input: bool = False
    status_byte: int = field(default=0, repr=False)

    @staticmethod
    def from_row(params, alpha, beta, nchi2, status, iters) -> "FitResult":
        p = [float(v) for v in params]
        # explicit5 rows carry (x, y, sigma, alpha, beta); alpha/beta also arrive separately
        shape = ShapeParams(*p[:3]) if len(p) in (3, 5) else EllipticalParams(*p)
        s = int(status)
        return FitResult(shape, Amplitudes(float(alpha), float(beta)), StopReason(s & 7), int(iters), float(nchi2),
                         bool(s & _lib.SF_FLAG_NOIMP), bool(s & _lib.SF_FLAG_INVALID), s)


def fit_single(image: SpotImage, init, config: FitConfig = FitConfig()) -> FitResult:
    """one spot through the GPU fitter (a batch of one;
    SPEC.md:387 "batch of 1 equals fit_single")."""
    from .batch_engine import fit_batch

    init_arr = np.asarray(init.as_array() if hasattr(init, "as_array") else init, dtype=np.float32)[None, :]
    res = fit_batch(image.values[None, :], inits=init_arr, config=config, grid=image.grid)
    return res[0]
