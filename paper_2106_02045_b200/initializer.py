"""Initial estimates on the GPU.

estimate_initial runs csrc/sf_init.cu (one warp per spot): 3x3 truncated
moving average, first argmax -> centre, min -> beta, max - beta -> alpha,
sigma = sqrt(M/pi) with M the count of original pixels above
alpha*exp(-0.5) + beta, clamped to the sigma bounds.
"""
from __future__ import annotations

import numpy as np

from .batch_engine import _as_image_array, estimate_initial_device
from .model import Amplitudes, EllipticalParams, ShapeParams, SpotImage
from .solver import FitConfig


def estimate_initial_batch(images, model: int = 3, config: FitConfig = FitConfig(), grid=None):
    """-> inits (count, model) f32, amps (count, 2) f32 [alpha, beta]."""
    import torch

    from . import _lib

    _lib.require_gpu()
    imgs, grid = _as_image_array(images, grid)
    # the initializer kernel reads float32 pixels: u16 counts (kept as u16 by _as_image_array for the
    # fit path) are widened exactly first
    t = imgs if isinstance(imgs, torch.Tensor) else torch.as_tensor(np.asarray(imgs, dtype=np.float32)).cuda()
    t = t.float().contiguous()
    ini, am = estimate_initial_device(t, grid, model, config, amps=True)
    torch.cuda.current_stream().synchronize()
    return ini.cpu().numpy(), am.cpu().numpy()


def estimate_initial(image: SpotImage, config: FitConfig = FitConfig(), model: int = 3):
    """-> (ShapeParams | EllipticalParams, Amplitudes)."""
    ini, am = estimate_initial_batch(image.values[None, :], model, config, grid=image.grid)
    shape = ShapeParams(*ini[0]) if model == 3 else EllipticalParams(*ini[0])
    return shape, Amplitudes(float(am[0, 0]), float(am[0, 1]))
