"""B200-native implicit-amplitude Levenberg-Marquardt fitter for 2D Gaussian
spots (arXiv 2106.02045), a drop-in for the reference's batch fit path.

Public API mirrors the reference package (pkg/src/spotfit/model.py and the
SPEC.md solver / batch_engine modules); the arithmetic runs in hand-written
sm_100a CUDA behind the C-ABI in include/spotfit.h.
"""
from .model import (MAX_PIXELS, DENOM_GUARD, Amplitudes, EllipticalParams, GradientSums, ModelEvaluation,
                    PixelGrid, ProfileSums, ShapeParams, SingularProfile, SpotImage, evaluate, evaluate_batch)
from .solver import FitConfig, FitResult, ParameterBounds, StopReason, fit_single
from .batch_engine import BatchRequest, BatchResult, fit_batch
from .simulator import SimConfig, simulate_batch, simulate_batch_device, simulate_spot
from .initializer import estimate_initial, estimate_initial_batch

__all__ = [
    "MAX_PIXELS", "DENOM_GUARD", "Amplitudes", "EllipticalParams", "GradientSums", "ModelEvaluation", "PixelGrid",
    "ProfileSums", "ShapeParams", "SingularProfile", "SpotImage", "evaluate", "evaluate_batch", "FitConfig",
    "FitResult", "ParameterBounds", "StopReason", "fit_single", "BatchRequest", "BatchResult", "fit_batch",
    "SimConfig", "simulate_batch", "simulate_batch_device", "simulate_spot", "estimate_initial",
    "estimate_initial_batch",
]
