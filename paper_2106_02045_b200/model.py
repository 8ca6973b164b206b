"""Model-level types and the batched model evaluation.

Mirrors the reference module ``spotfit.model`` (pkg/src/spotfit/model.py):
same type names, field meanings, float32 quantisation and error behaviour
(ValueError for bad grids, model.py:53-58,79-82,88-89; SingularProfile,
model.py:31-32).  The arithmetic of profile_and_gradient -> alpha_beta ->
chi_squared -> gradient_sums -> coefficient_gradients -> chi_gradient
(model.py:180-315) runs on the GPU through ``sf_eval_batch_device``
(include/spotfit.h), bit-identical to the reference.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MAX_PIXELS = 1024  # model.py:25
DENOM_GUARD = 1e-12  # model.py:28


class SingularProfile(ValueError):
    """The profile is numerically constant; amplitudes are not identifiable (model.py:31-32)."""


@dataclass(frozen=True)
class PixelGrid:
    """Row-major raster, pixel i at (i mod width, i div width) (model.py:44-67)."""

    width: int
    height: int

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ValueError(f"degenerate grid {self.width}x{self.height}")
        if self.width * self.height > MAX_PIXELS:
            raise ValueError(f"grid {self.width}x{self.height} exceeds {MAX_PIXELS} pixels")

    @property
    def n(self) -> int:
        return self.width * self.height

    @property
    def coords(self):
        i = np.arange(self.n)
        return (i % self.width).astype(np.float32), (i // self.width).astype(np.float32)


@dataclass(frozen=True)
class SpotImage:
    """One region of interest: grid + row-major float32 values (model.py:70-93)."""

    grid: PixelGrid
    values: np.ndarray

    def __post_init__(self):
        v = np.ascontiguousarray(np.asarray(self.values, dtype=np.float32).reshape(-1))
        if v.size != self.grid.n:
            raise ValueError(f"expected {self.grid.n} pixel values, got {v.size}")
        object.__setattr__(self, "values", v)

    @classmethod
    def from_array(cls, array) -> "SpotImage":
        a = np.asarray(array)
        if a.ndim != 2:
            raise ValueError("expected a 2D array")
        return cls(PixelGrid(a.shape[1], a.shape[0]), a)

    def as_2d(self) -> np.ndarray:
        return self.values.reshape(self.grid.height, self.grid.width)


def _f32(v) -> float:
    return float(np.float32(v))


@dataclass(frozen=True)
class ShapeParams:
    """(x, y, sigma) in pixels, quantised to float32 (model.py:100-115)."""

    x: float
    y: float
    sigma: float

    def __post_init__(self):
        object.__setattr__(self, "x", _f32(self.x))
        object.__setattr__(self, "y", _f32(self.y))
        object.__setattr__(self, "sigma", _f32(self.sigma))

    def as_array(self) -> np.ndarray:
        return np.array([self.x, self.y, self.sigma], dtype=np.float32)


@dataclass(frozen=True)
class EllipticalParams:
    """(x, y, sigma_x, sigma_y): the BASELINE config-3 model;
    the reference lists it as a non-goal, so no reference exists."""

    x: float
    y: float
    sigma_x: float
    sigma_y: float

    def __post_init__(self):
        for k in ("x", "y", "sigma_x", "sigma_y"):
            object.__setattr__(self, k, _f32(getattr(self, k)))

    def as_array(self) -> np.ndarray:
        return np.array([self.x, self.y, self.sigma_x, self.sigma_y], dtype=np.float32)


@dataclass(frozen=True)
class Amplitudes:
    """Implicit alpha, beta quantised to float32 (model.py:118-127)."""

    alpha: float
    beta: float

    def __post_init__(self):
        object.__setattr__(self, "alpha", _f32(self.alpha))
        object.__setattr__(self, "beta", _f32(self.beta))


@dataclass(frozen=True)
class ProfileSums:
    """model.py:130-140."""

    n: int
    f_sum: float
    g_sum: float
    ff_sum: float
    fg_sum: float
    denom: float


@dataclass(frozen=True)
class GradientSums:
    """model.py:143-151."""

    df: np.ndarray
    dff: np.ndarray
    dfg: np.ndarray
    gamma: np.ndarray


@dataclass(frozen=True)
class ModelEvaluation:
    """Everything the reference call chain produces for one (image, params):
    amps (alpha_beta), sums (ProfileSums), chi2 (chi_squared), gsums
    (gradient_sums), coefficient gradients, grad (chi_gradient, = -2 rhs),
    rhs and the upper-packed normal matrix jtj."""

    amps: Amplitudes
    sums: ProfileSums
    chi2: float
    gsums: GradientSums
    dalpha: np.ndarray
    dbeta: np.ndarray
    grad: np.ndarray
    rhs: np.ndarray
    jtj: np.ndarray


EVAL_DTYPE = np.dtype(
    [("singular", np.int32), ("alpha", np.float32), ("beta", np.float32), ("chi", np.float32), ("F", np.float64),
     ("G", np.float64), ("FF", np.float64), ("FG", np.float64), ("denom", np.float64), ("dF", np.float64, 4),
     ("dFF", np.float64, 4), ("dFG", np.float64, 4), ("gamma", np.float64, 4), ("dalpha", np.float64, 4),
     ("dbeta", np.float64, 4), ("rhs", np.float64, 4), ("jtj", np.float64, 10)],
    align=True,
)


def params_array(params) -> np.ndarray:
    """Accept ShapeParams / EllipticalParams / sequences / (count, P) arrays."""
    if isinstance(params, (ShapeParams, EllipticalParams)):
        return params.as_array()[None, :]
    if isinstance(params, (list, tuple)) and params and isinstance(params[0], (ShapeParams, EllipticalParams)):
        return np.stack([p.as_array() for p in params])
    a = np.asarray(params, dtype=np.float32)
    return a[None, :] if a.ndim == 1 else a


def evaluate_batch(images, params, width: int, height: int) -> np.ndarray:
    """GPU model evaluation for a batch: returns EVAL_DTYPE records (one per
    spot).  images: (count, H*W) or (count, H, W) float32; params: (count, P)."""
    import torch

    from . import _lib

    PixelGrid(width, height)
    _lib.require_gpu()
    imgs = torch.as_tensor(np.ascontiguousarray(images, np.float32).reshape(len(params), -1)).cuda()
    par = torch.as_tensor(np.ascontiguousarray(params, np.float32)).cuda()
    count, P = par.shape
    if imgs.shape[1] != width * height:
        raise ValueError(f"expected {width * height} pixel values per image, got {imgs.shape[1]}")
    out = torch.empty((count, EVAL_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().sf_eval_batch_device(imgs.data_ptr(), width, height, count, P, par.data_ptr(),
                                               out.data_ptr(), stream))
    torch.cuda.current_stream().synchronize()
    return out.cpu().numpy().view(EVAL_DTYPE).reshape(count)


def evaluate(image: SpotImage, params) -> ModelEvaluation:
    """One spot through the whole model chain (model.py:180-315) on the GPU.
    Raises SingularProfile exactly where alpha_beta would (model.py:228-231)."""
    p = params_array(params)
    r = evaluate_batch(image.values[None, :], p, image.grid.width, image.grid.height)[0]
    if r["singular"]:
        raise SingularProfile("constant profile: N*FF - F^2 not safely positive")
    P = p.shape[1]
    n = image.grid.n
    return ModelEvaluation(
        amps=Amplitudes(float(r["alpha"]), float(r["beta"])),
        sums=ProfileSums(n, float(r["F"]), float(r["G"]), float(r["FF"]), float(r["FG"]), float(r["denom"])),
        chi2=float(r["chi"]),
        gsums=GradientSums(r["dF"][:P].copy(), r["dFF"][:P].copy(), r["dFG"][:P].copy(), r["gamma"][:P].copy()),
        dalpha=r["dalpha"][:P].copy(),
        dbeta=r["dbeta"][:P].copy(),
        grad=-2.0 * r["rhs"][:P],
        rhs=r["rhs"][:P].copy(),
        jtj=r["jtj"][: P * (P + 1) // 2].copy(),
    )
