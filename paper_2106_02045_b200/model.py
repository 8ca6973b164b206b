"""Model-level types and the batched model evaluation.

Mirrors the reference module ``spotfit.model`` (pkg/src/spotfit/model.py):
same type names, field meanings, float32 quantisation and error behaviour
(ValueError for bad grids, model.py:53-58,79-82,88-89; SingularProfile,
model.py:31-32).  Every reference function -- profile, profile_and_gradient,
profile_gradient, alpha_beta, model_values, residuals, chi_squared,
gradient_sums, coefficient_gradients, chi_gradient (model.py:168-315) -- runs
on the GPU through the sf_model_* entry points (csrc/sf_model.cu), and the
whole chain at once through ``sf_eval_batch_device`` (evaluate /
evaluate_batch), bit-identical to the reference.
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


# ---------------------------------------------------------------------------------------------
# The spotfit.model function surface (model.py:168-315) on the GPU.  Each function keeps the
# reference's name, arguments, return types and errors; the arithmetic runs in sf_model.cu
# through the sf_model_* entry points (include/spotfit.h).  The *_batch forms take (count, ...)
# arrays (numpy or CUDA tensors) and return CUDA tensors; the reference-shaped single-spot
# forms wrap them.  There is no CPU fallback.
# ---------------------------------------------------------------------------------------------
def _cuda(a, dtype):
    import torch

    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(a))
    return t.to(device="cuda" if not t.is_cuda else t.device, dtype=dtype).contiguous()


def _stream():
    import torch

    return torch.cuda.current_stream().cuda_stream


def _model_of(P: int) -> int:
    if P not in (3, 4):
        raise ValueError(f"shape parameters must have 3 (x, y, sigma) or 4 (x, y, sigma_x, sigma_y) columns, got {P}")
    return P


def profile_batch(params, grid: PixelGrid, gradient: bool = False):
    """profile (model.py:168-177) / profile_and_gradient (180-199) for (count, P) params ->
    f (count, N) [, fgrad (count, N, P)] CUDA tensors."""
    import torch

    from . import _lib

    _lib.require_gpu()
    par = _cuda(params, torch.float32)
    par = par.reshape(1, -1) if par.dim() == 1 else par
    count, P = par.shape
    _model_of(P)
    f = torch.empty((count, grid.n), dtype=torch.float32, device=par.device)
    fg = torch.empty((count, grid.n, P), dtype=torch.float32, device=par.device) if gradient else None
    _lib.check(_lib.lib().sf_model_profile_device(par.data_ptr(), grid.width, grid.height, count, P, f.data_ptr(),
                                                  fg.data_ptr() if fg is not None else None, _stream()))
    return (f, fg) if gradient else f


def alpha_beta_batch(f, images):
    """alpha_beta (model.py:207-234) for (count, N) profiles and images -> alpha, beta (count,)
    f32 (NaN where SingularProfile), sums (count, 5) f64 = (F, G, FF, FG, denom), singular (count,)."""
    import torch

    from . import _lib

    _lib.require_gpu()
    ft, gt = _cuda(f, torch.float32), _cuda(images, torch.float32)
    count, n = ft.shape
    gt = gt.reshape(count, n)
    dev = ft.device
    a = torch.empty(count, dtype=torch.float32, device=dev)
    b = torch.empty(count, dtype=torch.float32, device=dev)
    sums = torch.empty((count, 5), dtype=torch.float64, device=dev)
    sing = torch.empty(count, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().sf_model_alpha_beta_device(ft.data_ptr(), gt.data_ptr(), n, count, a.data_ptr(),
                                                     b.data_ptr(), sums.data_ptr(), sing.data_ptr(), _stream()))
    return a, b, sums, sing


def chi_squared_batch(images, f, alpha, beta, values: bool = False):
    """model_values / residuals / chi_squared (model.py:237-250) -> chi (count,) f32
    [, h (count, N), r (count, N)]."""
    import torch

    from . import _lib

    _lib.require_gpu()
    ft = _cuda(f, torch.float32)
    count, n = ft.shape
    gt = _cuda(images, torch.float32).reshape(count, n)
    at, bt = _cuda(alpha, torch.float32).reshape(count), _cuda(beta, torch.float32).reshape(count)
    chi = torch.empty(count, dtype=torch.float32, device=ft.device)
    h = torch.empty((count, n), dtype=torch.float32, device=ft.device) if values else None
    r = torch.empty((count, n), dtype=torch.float32, device=ft.device) if values else None
    _lib.check(_lib.lib().sf_model_chi_squared_device(gt.data_ptr(), ft.data_ptr(), at.data_ptr(), bt.data_ptr(), n,
                                                      count, h.data_ptr() if values else None,
                                                      r.data_ptr() if values else None, chi.data_ptr(), _stream()))
    return (chi, h, r) if values else chi


def gradient_sums_batch(f, fgrad, images, sums):
    """gradient_sums (model.py:253-267) -> (count, 4, P) f64: df, dff, dfg, gamma."""
    import torch

    from . import _lib

    _lib.require_gpu()
    ft = _cuda(f, torch.float32)
    count, n = ft.shape
    fg = _cuda(fgrad, torch.float32).reshape(count, n, -1)
    P = _model_of(fg.shape[2])
    gt = _cuda(images, torch.float32).reshape(count, n)
    st = _cuda(sums, torch.float64).reshape(count, 5)
    out = torch.empty((count, 4, P), dtype=torch.float64, device=ft.device)
    _lib.check(_lib.lib().sf_model_gradient_sums_device(ft.data_ptr(), fg.data_ptr(), gt.data_ptr(), st.data_ptr(),
                                                        n, P, count, out.data_ptr(), _stream()))
    return out


def coefficient_gradients_batch(sums, gsums, alpha, beta, n: int):
    """coefficient_gradients (model.py:270-288) -> dalpha, dbeta (count, P) f64, singular (count,)."""
    import torch

    from . import _lib

    _lib.require_gpu()
    gs = _cuda(gsums, torch.float64)
    count, _, P = gs.shape
    _model_of(P)
    st = _cuda(sums, torch.float64).reshape(count, 5)
    at, bt = _cuda(alpha, torch.float32).reshape(count), _cuda(beta, torch.float32).reshape(count)
    da = torch.empty((count, P), dtype=torch.float64, device=gs.device)
    db = torch.empty((count, P), dtype=torch.float64, device=gs.device)
    sing = torch.empty(count, dtype=torch.int32, device=gs.device)
    _lib.check(_lib.lib().sf_model_coefficient_gradients_device(st.data_ptr(), gs.data_ptr(), at.data_ptr(),
                                                                bt.data_ptr(), n, P, count, da.data_ptr(),
                                                                db.data_ptr(), sing.data_ptr(), _stream()))
    return da, db, sing


def chi_gradient_batch(images, f, fgrad, alpha, beta, dalpha, dbeta):
    """chi_gradient (model.py:291-315) -> grad (count, P) f64, dmat (count, N, P) f32."""
    import torch

    from . import _lib

    _lib.require_gpu()
    ft = _cuda(f, torch.float32)
    count, n = ft.shape
    fg = _cuda(fgrad, torch.float32).reshape(count, n, -1)
    P = _model_of(fg.shape[2])
    gt = _cuda(images, torch.float32).reshape(count, n)
    at, bt = _cuda(alpha, torch.float32).reshape(count), _cuda(beta, torch.float32).reshape(count)
    da, db = _cuda(dalpha, torch.float64).reshape(count, P), _cuda(dbeta, torch.float64).reshape(count, P)
    grad = torch.empty((count, P), dtype=torch.float64, device=ft.device)
    dmat = torch.empty((count, n, P), dtype=torch.float32, device=ft.device)
    _lib.check(_lib.lib().sf_model_chi_gradient_device(gt.data_ptr(), ft.data_ptr(), fg.data_ptr(), at.data_ptr(),
                                                       bt.data_ptr(), da.data_ptr(), db.data_ptr(), n, P, count,
                                                       grad.data_ptr(), dmat.data_ptr(), _stream()))
    return grad, dmat


def _np(t):
    return t.cpu().numpy()


def _params_row(p) -> np.ndarray:
    if isinstance(p, (ShapeParams, EllipticalParams)):
        return p.as_array()
    return np.asarray(p, np.float32).reshape(-1)


def profile(p, grid: PixelGrid) -> np.ndarray:
    """model.py:168-177: unit-peak Gaussian profile f_i (float32, one numpy exp per pixel)."""
    return _np(profile_batch(_params_row(p)[None, :], grid))[0]


def profile_and_gradient(p, grid: PixelGrid):
    """model.py:180-199: (f, fgrad) with fgrad[:, j] = df/dp_j (x, y, sigma) -- or (x, y,
    sigma_x, sigma_y) for EllipticalParams."""
    f, fg = profile_batch(_params_row(p)[None, :], grid, gradient=True)
    return _np(f)[0], _np(fg)[0]


def profile_gradient(p, grid: PixelGrid) -> np.ndarray:
    """model.py:202-204."""
    return profile_and_gradient(p, grid)[1]


def alpha_beta(f, image: SpotImage):
    """model.py:207-234: closed-form amplitudes (Eq. 6) -> (Amplitudes, ProfileSums); raises
    SingularProfile where the reference does (denom <= DENOM_GUARD * N * FF)."""
    f = np.asarray(f, np.float32).reshape(-1)
    if f.size != image.grid.n:
        raise ValueError(f"expected {image.grid.n} profile values, got {f.size}")
    a, b, sums, sing = alpha_beta_batch(f[None, :], image.values[None, :])
    s = _np(sums)[0]
    ps = ProfileSums(f.size, float(s[0]), float(s[1]), float(s[2]), float(s[3]), float(s[4]))
    if int(_np(sing)[0]):
        raise SingularProfile(f"constant profile: N*FF - F^2 = {ps.denom:g} with N*FF = {f.size * ps.ff_sum:g}")
    return Amplitudes(float(_np(a)[0]), float(_np(b)[0])), ps


def _chi_parts(image: SpotImage, f, amps: Amplitudes):
    f = np.asarray(f, np.float32).reshape(-1)
    return chi_squared_batch(image.values[None, :], f[None, :], np.float32([amps.alpha]), np.float32([amps.beta]),
                             values=True)


def model_values(f, amps: Amplitudes) -> np.ndarray:
    """model.py:237-239: h_i = alpha*f_i + beta in float32."""
    f = np.asarray(f, np.float32).reshape(-1)
    _, h, _ = chi_squared_batch(np.zeros((1, f.size), np.float32), f[None, :], np.float32([amps.alpha]),
                                np.float32([amps.beta]), values=True)
    return _np(h)[0]


def residuals(image: SpotImage, f, amps: Amplitudes) -> np.ndarray:
    """model.py:242-244: r_i = g_i - (alpha*f_i + beta)."""
    return _np(_chi_parts(image, f, amps)[2])[0]


def chi_squared(image: SpotImage, f, amps: Amplitudes) -> float:
    """model.py:247-250: sum r_i^2 (float32 addends, float64 sum) quantised to float32."""
    return float(_np(_chi_parts(image, f, amps)[0])[0])


def gradient_sums(f, fgrad, image: SpotImage, sums: ProfileSums) -> GradientSums:
    """model.py:253-267."""
    f = np.asarray(f, np.float32).reshape(-1)
    s = np.array([[sums.f_sum, sums.g_sum, sums.ff_sum, sums.fg_sum, sums.denom]], np.float64)
    out = _np(gradient_sums_batch(f[None, :], np.asarray(fgrad, np.float32)[None], image.values[None, :], s))[0]
    return GradientSums(df=out[0].copy(), dff=out[1].copy(), dfg=out[2].copy(), gamma=out[3].copy())


def coefficient_gradients(sums: ProfileSums, gsums: GradientSums, amps: Amplitudes):
    """model.py:270-288: (dalpha, dbeta), Eq. (8); raises SingularProfile like the reference."""
    s = np.array([[sums.f_sum, sums.g_sum, sums.ff_sum, sums.fg_sum, sums.denom]], np.float64)
    g = np.stack([gsums.df, gsums.dff, gsums.dfg, gsums.gamma])[None].astype(np.float64)
    da, db, sing = coefficient_gradients_batch(s, g, np.float32([amps.alpha]), np.float32([amps.beta]), sums.n)
    if int(_np(sing)[0]):
        raise SingularProfile("constant profile: amplitude gradients undefined")
    return _np(da)[0], _np(db)[0]


def chi_gradient(image: SpotImage, f, fgrad, amps: Amplitudes, coeff_grads):
    """model.py:291-315: (grad, dmat), Eq. (9); grad_j = -2 sum r_i d_ij."""
    da, db = coeff_grads
    f = np.asarray(f, np.float32).reshape(-1)
    grad, dmat = chi_gradient_batch(image.values[None, :], f[None, :], np.asarray(fgrad, np.float32)[None],
                                    np.float32([amps.alpha]), np.float32([amps.beta]),
                                    np.asarray(da, np.float64)[None], np.asarray(db, np.float64)[None])
    return _np(grad)[0], _np(dmat)[0]


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
