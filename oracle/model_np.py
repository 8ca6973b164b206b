"""numpy restatement of the reference model arithmetic (TEST INFRASTRUCTURE ONLY).

Restates /root/reference/pkg/src/spotfit/model.py so that the oracle travels to
the GPU box (where /root/reference does not exist).  Same numeric contract as
the reference (model.py:11-14): float32 per-pixel values and products, float64
pairwise reductions via ``ndarray.sum(dtype=float64)``, float32 quantisation of
shape, amplitudes and chi^2.  The function names are the reference's so the LM
loop in oracle/lm.py can run over either module; tests/test_oracle_golden.py
pins every function bit-for-bit against fixtures produced by the reference
itself (tests/golden/make_golden.py).

Also holds the elliptical (x0, y0, sx, sy) extension of SURVEY.md App. B.5,
which has no reference counterpart -- parity unpinned there.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

MAX_PIXELS = 1024  # model.py:25
DENOM_GUARD = 1e-12  # model.py:28
_F64 = np.float64
_F32 = np.float32


class SingularProfile(ValueError):
    """model.py:31-32 -- N*FF - F^2 not safely positive."""


@lru_cache(maxsize=256)
def _coords(width: int, height: int):
    # model.py:35-41: row-major, x = i mod W, y = i div W, origin at pixel 0
    idx = np.arange(width * height)
    x = (idx % width).astype(_F32)
    y = (idx // width).astype(_F32)
    x.flags.writeable = False
    y.flags.writeable = False
    return x, y


@dataclass(frozen=True)
class PixelGrid:  # model.py:44-67
    width: int
    height: int

    def __post_init__(self):
        if min(self.width, self.height) < 1:
            raise ValueError(f"degenerate grid {self.width}x{self.height}")
        if self.width * self.height > MAX_PIXELS:
            raise ValueError(f"grid {self.width}x{self.height} exceeds {MAX_PIXELS} pixels")

    @property
    def n(self) -> int:
        return self.width * self.height

    @property
    def coords(self):
        return _coords(self.width, self.height)


@dataclass(frozen=True)
class SpotImage:  # model.py:70-93
    grid: PixelGrid
    values: np.ndarray

    def __post_init__(self):
        flat = np.ascontiguousarray(np.asarray(self.values, dtype=_F32).reshape(-1))
        if flat.size != self.grid.n:
            raise ValueError(f"expected {self.grid.n} pixel values, got {flat.size}")
        object.__setattr__(self, "values", flat)

    @classmethod
    def from_array(cls, array):
        a = np.asarray(array)
        if a.ndim != 2:
            raise ValueError("expected a 2D array")
        return cls(PixelGrid(a.shape[1], a.shape[0]), a)


def _q32(v) -> float:
    return float(_F32(v))


@dataclass(frozen=True)
class ShapeParams:  # model.py:100-115 -- quantised to f32 on construction
    x: float
    y: float
    sigma: float

    def __post_init__(self):
        for k in ("x", "y", "sigma"):
            object.__setattr__(self, k, _q32(getattr(self, k)))

    def as_array(self):
        return np.array([self.x, self.y, self.sigma], dtype=_F32)


@dataclass(frozen=True)
class EllipticalParams:  # SURVEY App. B.5 (no reference)
    x: float
    y: float
    sigma_x: float
    sigma_y: float

    def __post_init__(self):
        for k in ("x", "y", "sigma_x", "sigma_y"):
            object.__setattr__(self, k, _q32(getattr(self, k)))

    def as_array(self):
        return np.array([self.x, self.y, self.sigma_x, self.sigma_y], dtype=_F32)


@dataclass(frozen=True)
class Amplitudes:  # model.py:118-127
    alpha: float
    beta: float

    def __post_init__(self):
        object.__setattr__(self, "alpha", _q32(self.alpha))
        object.__setattr__(self, "beta", _q32(self.beta))


@dataclass(frozen=True)
class ProfileSums:  # model.py:130-140
    n: int
    f_sum: float
    g_sum: float
    ff_sum: float
    fg_sum: float
    denom: float


@dataclass(frozen=True)
class GradientSums:  # model.py:143-151
    df: np.ndarray
    dff: np.ndarray
    dfg: np.ndarray
    gamma: np.ndarray


def _offsets(p, grid: PixelGrid):
    """model.py:154-165 (and App. B.5 for EllipticalParams): one IEEE f32
    reciprocal per axis, then multiplications only."""
    x, y = grid.coords
    if isinstance(p, EllipticalParams):
        ix = _F32(1.0) / _F32(p.sigma_x)
        iy = _F32(1.0) / _F32(p.sigma_y)
    else:
        ix = iy = _F32(1.0) / _F32(p.sigma)
    return (x - _F32(p.x)) * ix, (y - _F32(p.y)) * iy, ix, iy


def profile(p, grid: PixelGrid) -> np.ndarray:
    """model.py:168-177."""
    u, v, _, _ = _offsets(p, grid)
    return np.exp(_F32(-0.5) * (u * u + v * v))


def profile_and_gradient(p, grid: PixelGrid):
    """model.py:180-199 for ShapeParams (columns x, y, sigma); App. B.5 for
    EllipticalParams (columns x, y, sigma_x, sigma_y)."""
    u, v, ix, iy = _offsets(p, grid)
    q = u * u + v * v
    f = np.exp(_F32(-0.5) * q)
    if isinstance(p, EllipticalParams):
        dx = u * (f * ix)
        dy = v * (f * iy)
        cols = (dx, dy, u * dx, v * dy)
    else:
        fs = f * ix
        cols = (u * fs, v * fs, q * fs)
    return f, np.stack(cols, axis=1).astype(_F32, copy=False)


def profile_gradient(p, grid: PixelGrid):
    return profile_and_gradient(p, grid)[1]  # model.py:202-204


def _sum64(a) -> float:
    return float(a.sum(dtype=_F64))


def alpha_beta(f, image: SpotImage):
    """model.py:207-234: Eq. (6) with the relative singularity guard."""
    g = image.values
    n = f.size
    F, G = _sum64(f), _sum64(g)
    FF, FG = _sum64(f * f), _sum64(f * g)
    denom = n * FF - F * F
    sums = ProfileSums(n, F, G, FF, FG, denom)
    if denom <= DENOM_GUARD * n * FF:
        raise SingularProfile(f"constant profile: N*FF - F^2 = {denom:g}")
    return Amplitudes((n * FG - F * G) / denom, (G * FF - F * FG) / denom), sums


def model_values(f, amps: Amplitudes):
    return _F32(amps.alpha) * f + _F32(amps.beta)  # model.py:237-239


def residuals(image: SpotImage, f, amps: Amplitudes):
    return image.values - model_values(f, amps)  # model.py:242-244


def chi_squared(image: SpotImage, f, amps: Amplitudes) -> float:
    r = residuals(image, f, amps)  # model.py:247-250
    return _q32(_sum64(r * r))


def gradient_sums(f, fgrad, image: SpotImage, sums: ProfileSums) -> GradientSums:
    """model.py:253-267 (column count = number of shape parameters)."""
    g = image.values
    P = fgrad.shape[1]
    df = np.array([_sum64(fgrad[:, j]) for j in range(P)])
    dff = np.array([2.0 * _sum64(f * fgrad[:, j]) for j in range(P)])
    dfg = np.array([_sum64(g * fgrad[:, j]) for j in range(P)])
    return GradientSums(df, dff, dfg, sums.n * dff - 2.0 * sums.f_sum * df)


def coefficient_gradients(sums: ProfileSums, gs: GradientSums, amps: Amplitudes):
    """model.py:270-288: Eq. (8)."""
    if sums.denom <= DENOM_GUARD * sums.n * sums.ff_sum:
        raise SingularProfile("constant profile: amplitude gradients undefined")
    D = sums.denom
    da = (sums.n * gs.dfg - sums.g_sum * gs.df - amps.alpha * gs.gamma) / D
    db = (sums.g_sum * gs.dff - sums.fg_sum * gs.df - sums.f_sum * gs.dfg - amps.beta * gs.gamma) / D
    return da, db


def chi_gradient(image: SpotImage, f, fgrad, amps: Amplitudes, coeff_grads):
    """model.py:291-315: Eq. (9); returns (grad, d) with d_ij the per-pixel
    model derivative, grad_j = -2 * sum r_i d_ij."""
    da, db = coeff_grads
    r = residuals(image, f, amps)
    a32 = _F32(amps.alpha)
    P = fgrad.shape[1]
    d = np.empty_like(fgrad)
    for j in range(P):
        d[:, j] = _F32(da[j]) * f + a32 * fgrad[:, j] + _F32(db[j])
    grad = np.array([-2.0 * _sum64(r * d[:, j]) for j in range(P)])
    return grad, d
