"""Synthetic spots through sf_simulate_host.

Counter-based Philox4x32-10 keyed by (seed, index): any index regenerates
alone, and generation is independent of thread count.
Test/bench input generator -- not on the timed path.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class SimConfig:
    """SPEC.md:321-324 (defaults: 400 signal, 40 background counts, sigma in [1, 2])."""

    width: int = 9
    height: int = 9
    count: int = 1
    n_signal: float = 400.0
    n_background: float = 40.0
    sigma_range: tuple = (1.0, 2.0)
    center_spread: float = 0.0  # <= 0: S/20 per axis
    noise: bool = True
    rounding: bool = True
    seed: int = 0
    model: int = 3  # 4: independent sigma_x, sigma_y (BASELINE config 3)

    def to_c(self) -> _lib.sf_sim_config:
        return _lib.sf_sim_config(self.model, self.n_signal, self.n_background, self.sigma_range[0],
                                  self.sigma_range[1], self.center_spread, int(self.noise), int(self.rounding),
                                  self.seed & 0xFFFFFFFFFFFFFFFF)


def simulate_batch(cfg: SimConfig, first_index: int = 0, threads: int = 0):
    """-> images (count, H, W) f32, truth (count, P+2) f32 [x, y, sigma(s), alpha, beta]."""
    N = cfg.width * cfg.height
    images = np.empty((cfg.count, cfg.height, cfg.width), np.float32)
    truth = np.empty((cfg.count, cfg.model + 2), np.float32)
    c = cfg.to_c()
    rc = _lib.lib().sf_simulate_host(ctypes.byref(c), cfg.width, cfg.height, first_index, cfg.count,
                                     images.ctypes.data, truth.ctypes.data, threads)
    if rc != 0:
        raise ValueError("invalid simulation config")
    assert images.size == cfg.count * N
    return images, truth


def simulate_batch_device(cfg: SimConfig, first_index: int = 0, device=None):
    """The generator on the GPU (sf_simulate_device): -> (images (count, H, W),
    truth (count, P+2)) as CUDA tensors, generated in HBM (no PCIe)."""
    import torch

    _lib.require_gpu()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    images = torch.empty((cfg.count, cfg.height, cfg.width), dtype=torch.float32, device=dev)
    truth = torch.empty((cfg.count, cfg.model + 2), dtype=torch.float32, device=dev)
    c = cfg.to_c()
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.lib().sf_simulate_device(ctypes.byref(c), cfg.width, cfg.height, first_index, cfg.count,
                                             images.data_ptr(), truth.data_ptr(), stream))
    return images, truth


def simulate_spot(cfg: SimConfig, index: int):
    """One spot by index: equals simulate_batch(...)[index]."""
    one = SimConfig(**{**cfg.__dict__, "count": 1})
    im, tr = simulate_batch(one, first_index=index, threads=1)
    return im[0], tr[0]
