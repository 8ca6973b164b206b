"""B200-native implicit-amplitude Levenberg-Marquardt fitter for 2D Gaussian
spots (arXiv 2106.02045), a drop-in for the reference's batch fit path.

Public API mirrors the reference package (pkg/src/spotfit/model.py and the
SPEC.md solver / batch_engine modules); the arithmetic runs in hand-written
sm_100a CUDA behind the C-ABI in include/spotfit.h.
"""
from .model import (MAX_PIXELS, DENOM_GUARD, Amplitudes, EllipticalParams, GradientSums, ModelEvaluation,
                    PixelGrid, ProfileSums, ShapeParams, SingularProfile, SpotImage, alpha_beta, alpha_beta_batch,
                    chi_gradient, chi_gradient_batch, chi_squared, chi_squared_batch, coefficient_gradients,
                    coefficient_gradients_batch, evaluate, evaluate_batch, gradient_sums, gradient_sums_batch,
                    model_values, profile, profile_and_gradient, profile_batch, profile_gradient, residuals)
from .solver import FitConfig, FitResult, ParameterBounds, StopReason, fit_single
from .batch_engine import BatchRequest, BatchResult, fit_batch
from .simulator import SimConfig, simulate_batch, simulate_batch_device, simulate_spot
from .initializer import estimate_initial, estimate_initial_batch

__all__ = [
    "MAX_PIXELS", "DENOM_GUARD", "Amplitudes", "EllipticalParams", "GradientSums", "ModelEvaluation", "PixelGrid",
    "ProfileSums", "ShapeParams", "SingularProfile", "SpotImage", "evaluate", "evaluate_batch", "profile",
    "profile_and_gradient", "profile_gradient", "alpha_beta", "model_values", "residuals", "chi_squared",
    "gradient_sums", "coefficient_gradients", "chi_gradient", "profile_batch", "alpha_beta_batch",
    "chi_squared_batch", "gradient_sums_batch", "coefficient_gradients_batch", "chi_gradient_batch", "FitConfig",
    "FitResult", "ParameterBounds", "StopReason", "fit_single", "BatchRequest", "BatchResult", "fit_batch",
    "SimConfig", "simulate_batch", "simulate_batch_device", "simulate_spot", "estimate_initial",
    "estimate_initial_batch",
]
