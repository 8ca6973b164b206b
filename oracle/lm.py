"""Restated LM solver and batch loop (TEST INFRASTRUCTURE ONLY).

The reference ships no solver code: the state machine below is
PAPER.md:126-180 (Fit2DGaussian pseudo-code) with SPEC.md:158-262 and the
resolutions pinned in SURVEY.md App. A / DESIGN.md section 3.  It runs over any
module exposing the reference model API (``spotfit.model`` itself when
/root/reference is importable -- tests/golden/make_golden.py does that -- or
oracle/model_np.py, the travelling restatement).  The C twin is
oracle/spotfit_oracle.c:sf_oracle_fit; tests pin the two against each other and
against the golden fixtures bit-for-bit.

This module is also the "reference CPU fitter" timed by bench.py --impl
reference: numpy per-call arithmetic exactly as the reference performs it.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

# StopReason codes; identical to include/spotfit.h
MAX_ERROR, MIN_DELTA, MIN_STEP, NOT_CONVERGED, MAX_ITERATIONS = range(5)
FLAG_INVALID = 0x40
FLAG_NOIMP = 0x80
STEP_GUARD = 1e-12  # SPEC.md:193, pinned


@dataclass(frozen=True)
class LMConfig:
    """FitConfig + ParameterBounds (defaults)."""

    max_iterations: int = 20
    max_error: float = 0.0
    min_delta: float = 1e-6
    min_step: float = 1e-4
    lambda_init: float = 0.01
    lambda_up: float = 10.0
    lambda_down: float = 10.0
    lambda_max: float = 1e4
    margin_x: float = 0.0
    margin_y: float = 0.0
    sigma_min: float = 0.3
    sigma_max: float = 0.0

    @staticmethod
    def for_grid(width: int, height: int, **kw) -> "LMConfig":
        base = dict(margin_x=width / 2, margin_y=height / 2, sigma_min=0.3, sigma_max=float(max(width, height)))
        base.update(kw)
        return LMConfig(**base)


def _clamp(v: float, lo: float, hi: float) -> float:
    return lo if v < lo else (hi if v > hi else v)


def limit(v, W: int, H: int, c: LMConfig) -> list:
    """clamp in f64, then quantise to f32 once (App. A [A4]).
    Explicit-5 (len 5): sigma free in sign with |sigma| bounded, alpha/beta free."""
    out = [_clamp(v[0], -c.margin_x, (W - 1) + c.margin_x), _clamp(v[1], -c.margin_y, (H - 1) + c.margin_y)]
    if len(v) == 5:
        s = v[2]
        out += [-_clamp(-s, c.sigma_min, c.sigma_max) if s < 0 else _clamp(s, c.sigma_min, c.sigma_max), v[3], v[4]]
    else:
        out += [_clamp(s, c.sigma_min, c.sigma_max) for s in v[2:]]
    return [float(np.float32(t)) for t in out]


def solve_pivot5(jtj_packed, rhs, lam: float):
    """Explicit-5 step: damped 5x5 system by Gaussian elimination
    with partial pivoting, f64, no FMA; None on StepFailed (zero pivot or
    |det| <= 1e-12 * prod(damped diagonal)).  Twin of spotfit_oracle.c:solve_pivot5."""
    P = 5
    M = [[0.0] * P for _ in range(P)]
    m = 0
    for i in range(P):
        for j in range(i, P):
            M[i][j] = M[j][i] = float(jtj_packed[m])
            m += 1
    b = [float(x) for x in rhs]
    for i in range(P):
        M[i][i] = M[i][i] + lam * M[i][i]
    dprod = M[0][0]
    for i in range(1, P):
        dprod = dprod * M[i][i]
    det = 1.0
    for col in range(P):
        pr, best = col, abs(M[col][col])
        for r in range(col + 1, P):
            if abs(M[r][col]) > best:
                best, pr = abs(M[r][col]), r
        if not (best > 0.0):
            return None
        if pr != col:
            M[col], M[pr] = M[pr], M[col]
            b[col], b[pr] = b[pr], b[col]
        det = det * M[col][col]
        for r in range(col + 1, P):
            fct = M[r][col] / M[col][col]
            for c in range(col, P):
                M[r][c] = M[r][c] - fct * M[col][c]
            b[r] = b[r] - fct * b[col]
    if not (abs(det) > STEP_GUARD * abs(dprod)):
        return None
    delta = [0.0] * P
    for r in reversed(range(P)):
        s = b[r]
        for c in range(r + 1, P):
            s = s - M[r][c] * delta[c]
        delta[r] = s / M[r][r]
    return delta


def solve_step(jtj_packed, rhs, lam: float):
    """Damped LDL^T solve of (JtJ + lam diag JtJ) delta = rhs (Eq. 12-14).

    f64, no FMA, fixed operation order (identical in spotfit_oracle.c and the
    CUDA kernel).  Returns None on StepFailed: a non-positive pivot or
    det <= 1e-12 * prod(damped diagonal)."""
    P = len(rhs)
    if P == 5:
        return solve_pivot5(jtj_packed, rhs, lam)
    A = [[0.0] * P for _ in range(P)]
    m = 0
    for i in range(P):
        for j in range(i, P):
            A[i][j] = A[j][i] = float(jtj_packed[m])
            m += 1
    for i in range(P):
        A[i][i] = A[i][i] + lam * A[i][i]
    L = [[0.0] * P for _ in range(P)]
    C = [[0.0] * P for _ in range(P)]
    D = [0.0] * P
    for i in range(P):
        for j in range(i):
            s = A[i][j]
            for k in range(j):
                s = s - C[i][k] * L[j][k]
            C[i][j] = s
            L[i][j] = s / D[j]
        s = A[i][i]
        for k in range(i):
            s = s - C[i][k] * L[i][k]
        D[i] = s
        if not (s > 0.0):
            return None
    det, dprod = D[0], A[0][0]
    for i in range(1, P):
        det = det * D[i]
        dprod = dprod * A[i][i]
    if not (det > STEP_GUARD * dprod):
        return None
    z = [0.0] * P
    for i in range(P):
        s = float(rhs[i])
        for k in range(i):
            s = s - L[i][k] * z[k]
        z[i] = s
    z = [z[i] / D[i] for i in range(P)]
    delta = [0.0] * P
    for i in reversed(range(P)):
        s = z[i]
        for k in range(i + 1, P):
            s = s - L[k][i] * delta[k]
        delta[i] = s
    return delta


class _Eval:
    __slots__ = ("singular", "chi", "alpha", "beta", "jtj", "rhs")


def _params(m, p):
    if len(p) == 4:
        return m.EllipticalParams(*p)
    return m.ShapeParams(*p)


def explicit5_eval(m, image, p) -> _Eval:
    """Explicit 5-parameter model, p = (x, y, sigma, alpha, beta):
    h = alpha*f + beta, d = (alpha*df/dx, alpha*df/dy, alpha*df/dsigma, f, 1) in f32,
    chi^2 / rhs / JtJ as f64 numpy-order sums of f32 products."""
    e = _Eval()
    f, fg = m.profile_and_gradient(m.ShapeParams(*p[:3]), image.grid)
    a32, b32 = np.float32(p[3]), np.float32(p[4])
    g = image.values
    r = g - (a32 * f + b32)
    d = [a32 * fg[:, 0], a32 * fg[:, 1], a32 * fg[:, 2], f, np.ones_like(f)]
    e.singular = False
    e.chi = float(np.float32((r * r).sum(dtype=np.float64)))
    e.alpha, e.beta = float(a32), float(b32)
    e.rhs = [float((r * dj).sum(dtype=np.float64)) for dj in d]
    e.jtj = [float((d[j] * d[k]).sum(dtype=np.float64)) for j in range(5) for k in range(j, 5)]
    return e


def g_eval(m, image, p) -> _Eval:
    """PAPER.md:139 Gaussian2D(..., gradient=true): chi^2, JtJ and rhs = Jt r."""
    if len(p) == 5:
        return explicit5_eval(m, image, p)
    e = _Eval()
    f, fg = m.profile_and_gradient(_params(m, p), image.grid)
    try:
        amps, sums = m.alpha_beta(f, image)
    except m.SingularProfile:
        e.singular, e.chi = True, math.nan
        return e
    e.singular = False
    e.chi = m.chi_squared(image, f, amps)
    e.alpha, e.beta = amps.alpha, amps.beta
    gs = m.gradient_sums(f, fg, image, sums)
    cg = m.coefficient_gradients(sums, gs, amps)
    grad, d = m.chi_gradient(image, f, fg, amps, cg)
    P = d.shape[1]
    e.rhs = [float(g) * -0.5 for g in grad]  # rhs_j = sum r*d_j = -grad_j/2 (exact)
    e.jtj = [float((d[:, j] * d[:, k]).sum(dtype=np.float64)) for j in range(P) for k in range(j, P)]
    return e


def t_eval(m, image, p) -> _Eval:
    """PAPER.md:151 Gaussian2D(..., gradient=false): profile -> alpha_beta -> chi^2."""
    if len(p) == 5:
        return explicit5_eval(m, image, p)
    e = _Eval()
    f = m.profile(_params(m, p), image.grid)
    try:
        amps, _ = m.alpha_beta(f, image)
    except m.SingularProfile:
        e.singular, e.chi = True, math.nan
        return e
    e.singular = False
    e.chi = m.chi_squared(image, f, amps)
    e.alpha, e.beta = amps.alpha, amps.beta
    return e


def fit_single(m, image, init, cfg: LMConfig) -> dict:
    """SURVEY.md App. A.  Returns params, alpha, beta, nchi2, status, iterations
    and the evaluation counts (n_g, n_t) used by the roofline accounting."""
    W, H = image.grid.width, image.grid.height
    N = W * H
    P = len(init)
    if not (np.all(np.isfinite(image.values)) and all(math.isfinite(float(v)) for v in init)):
        return dict(params=[float(np.float32(v)) for v in init], alpha=math.nan, beta=math.nan, nchi2=math.nan,
                    status=NOT_CONVERGED | FLAG_INVALID, iterations=0, n_g=0, n_t=0)
    p = limit([float(np.float32(v)) for v in init], W, H, cfg)
    lam = cfg.lambda_init
    it, stop, noimp, n_g, n_t = 0, MAX_ITERATIONS, 0, 0, 0
    fin_p, fin_e = p, None
    while it < cfg.max_iterations:
        it += 1
        eb = g_eval(m, image, p)
        n_g += 1
        if eb.singular or not math.isfinite(eb.chi):
            stop, fin_p, fin_e = NOT_CONVERGED, p, eb
            break
        if eb.chi < cfg.max_error:
            stop, fin_p, fin_e = MAX_ERROR, p, eb
            break
        chib, best = eb.chi, p
        thr = [cfg.min_step * max(abs(b), 1.0) for b in best]

        def trial():
            nonlocal n_t
            delta = solve_step(eb.jtj, eb.rhs, lam)
            if delta is None:  # StepFailed: like a non-decreasing step
                return math.inf, False, None, None
            tp = limit([b + d for b, d in zip(best, delta)], W, H, cfg)
            et = t_eval(m, image, tp)
            n_t += 1
            small = all(abs(d) < t for d, t in zip(delta, thr))
            return (math.nan if et.singular else et.chi), small, tp, et

        chit, small, tp, et = trial()
        if chib > chit:
            lam = lam / cfg.lambda_down
        while (not small) and chib < chit and lam < cfg.lambda_max:
            lam = lam * cfg.lambda_up
            chit, small, tp, et = trial()
        if math.isnan(chit) or (chib < chit and lam >= cfg.lambda_max):
            stop, fin_p, fin_e = NOT_CONVERGED, best, eb
            break
        if chib < chit:  # App. A [A2]
            stop, noimp, fin_p, fin_e = MIN_DELTA, 1, best, eb
            break
        p, fin_p, fin_e = tp, tp, et
        if chit < cfg.max_error:
            stop = MAX_ERROR
            break
        if chib * (1.0 - cfg.min_delta) < chit:
            stop = MIN_DELTA
            break
        if small:
            stop = MIN_STEP
            break
    if fin_e.singular:
        alpha = beta = nchi2 = math.nan
    else:
        alpha, beta = fin_e.alpha, fin_e.beta
        nchi2 = float(np.float32(fin_e.chi / (N - 5))) if N > 5 else fin_e.chi
    return dict(params=list(fin_p), alpha=alpha, beta=beta, nchi2=nchi2, status=stop | (FLAG_NOIMP if noimp else 0),
                iterations=it, n_g=n_g, n_t=n_t)


def fit_batch_arrays(m, images: np.ndarray, inits: np.ndarray, W: int, H: int, cfg: LMConfig) -> dict:
    """Sequential batch over (count, H*W) images; SoA result arrays."""
    count, P = inits.shape
    grid = m.PixelGrid(W, H)
    out = dict(params=np.zeros((count, P), np.float32), alpha=np.zeros(count, np.float32),
               beta=np.zeros(count, np.float32), nchi2=np.zeros(count, np.float32),
               status=np.zeros(count, np.uint8), iterations=np.zeros(count, np.uint8),
               n_g=np.zeros(count, np.int32), n_t=np.zeros(count, np.int32))
    for s in range(count):
        r = fit_single(m, m.SpotImage(grid, images[s].reshape(-1)), [float(v) for v in inits[s]], cfg)
        out["params"][s] = r["params"]
        for k in ("alpha", "beta", "nchi2", "status", "iterations", "n_g", "n_t"):
            out[k][s] = r[k]
    return out


REF_INSTALL = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def model_backend(name: str = "auto"):
    """The arithmetic under the LM loop: the unmodified reference ``spotfit.model``
    pip-installed into baseline/_ref when present ("reference"),
    else the restatement oracle/model_np.py ("port").  Returns (module, kind)."""
    if name in ("auto", "reference"):
        import sys

        if os.path.isdir(os.path.join(REF_INSTALL, "spotfit")):
            if REF_INSTALL not in sys.path:
                sys.path.insert(0, REF_INSTALL)
            from spotfit import model as ref_model

            return ref_model, "reference"
        if name == "reference":
            raise ImportError(f"reference spotfit not installed under {REF_INSTALL}")
    from oracle import model_np

    return model_np, "port"


def _worker(args):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    images, inits, W, H, cfg, backend = args
    m, _ = model_backend(backend)
    return fit_batch_arrays(m, images, inits, W, H, cfg)


_POOLS = {}


def _pool(workers: int):
    """Persistent worker pool (process start-up stays out of timed batches)."""
    import multiprocessing as mp

    if workers not in _POOLS:
        _POOLS[workers] = mp.get_context("fork").Pool(workers)
    return _POOLS[workers]


def fit_batch_parallel(images: np.ndarray, inits: np.ndarray, W: int, H: int, cfg: LMConfig, workers: int = 0,
                       backend: str = "auto"):
    """contiguous chunks over a process pool, order preserved."""
    workers = workers or len(os.sched_getaffinity(0))
    count = inits.shape[0]
    bounds = [(count * w // workers, count * (w + 1) // workers) for w in range(workers)]
    chunks = [(images[a:b], inits[a:b], W, H, cfg, backend) for a, b in bounds if b > a]
    parts = _pool(workers).map(_worker, chunks)
    return {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
