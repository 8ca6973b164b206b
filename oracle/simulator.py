"""Restated synthetic-spot generator (TEST / BENCH INFRASTRUCTURE ONLY).

SPEC.md:316-368 (simulate_spot / simulate_batch), with the
draws pinned exactly as the product's generator (csrc/sf_sim_core.h) makes them:
counter-based Philox4x32-10 keyed by the 64-bit seed with counter
(index lo, index hi, block, "SPOT"), uniforms (x + 0.5) 2^-32, Box-Muller
normals; block 0 -> centre offsets + sigma(s), block 1 + i/4 -> the noise
normals of pixels 4k..4k+3;
  lambda_i = alpha exp(-(dx^2 / (2 sx^2) + dy^2 / (2 sy^2))) + beta   (f64)
  g_i      = max(0, round_half_away(lambda_i + z_i sqrt(lambda_i)))  (f32).

Vectorised numpy over a whole batch, so ``bench.py --impl reference`` builds its
inputs without loading the product library.  numpy's float64 exp/log/sin/cos may
differ from glibc's in the last ulp; an integer pixel or an f32 truth value can
only change if such an ulp straddles a rounding boundary (probability ~1e-13
per pixel, ~2^-29 per value), and ``tests/test_simulator.py`` checks the two
generators bitwise on every spot of a sample.
"""
from __future__ import annotations

import numpy as np

M32 = np.uint64(0xFFFFFFFF)
TAG = 0x53504F54  # "SPOT"
TWO_PI = 6.283185307179586


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x32-10 on uint64 arrays holding 32-bit lanes (sf_sim_core.h:philox4x32_10)."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & M32 for c in (c0, c1, c2, c3))
    k0, k1 = np.uint64(k0 & 0xFFFFFFFF), np.uint64(k1 & 0xFFFFFFFF)
    for _ in range(10):
        p0 = np.uint64(0xD2511F53) * c0
        p1 = np.uint64(0xCD9E8D57) * c2
        n0 = (p1 >> np.uint64(32)) ^ c1 ^ k0
        n2 = (p0 >> np.uint64(32)) ^ c3 ^ k1
        c0, c1, c2, c3 = n0 & M32, p1 & M32, n2 & M32, p0 & M32
        k0 = (k0 + np.uint64(0x9E3779B9)) & M32
        k1 = (k1 + np.uint64(0xBB67AE85)) & M32
    return c0, c1, c2, c3


def block_uniforms(seed: int, index, blk):
    """-> u[4] f64 arrays broadcast over (index, blk): (x + 0.5) 2^-32."""
    index = np.asarray(index, dtype=np.int64).astype(np.uint64)
    blk = np.asarray(blk, dtype=np.uint64)
    index, blk = np.broadcast_arrays(index, blk)
    c = philox4x32_10(index & M32, index >> np.uint64(32), blk, np.full(index.shape, TAG, np.uint64),
                      seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    return [(x.astype(np.float64) + 0.5) * 2.3283064365386963e-10 for x in c]


def box_muller(u1, u2):
    r = np.sqrt(-2.0 * np.log(u1))
    t = TWO_PI * u2
    return r * np.cos(t), r * np.sin(t)


def _round_half_away(v):
    t = np.trunc(v)
    return t + np.where(np.abs(v - t) >= 0.5, np.sign(v), 0.0)


def unrounded(W: int, H: int, index: int, seed: int, model: int = 3, **kw):
    """The f64 value lambda_i + z_i sqrt(lambda_i) of every pixel of one spot before rounding and
    clamping -- tells a .5-boundary case (where two libms may round differently) from a real
    mismatch."""
    kw = dict(kw, rounding=False)
    return _values(W, H, 1, seed, model, index, **kw)[0][0]


def _values(W, H, count, seed, model, first_index, n_signal=400.0, n_background=40.0, sigma_lo=1.0, sigma_hi=2.0,
            spread=0.0, noise=True, rounding=True, clamp=False):
    seed &= 0xFFFFFFFFFFFFFFFF
    N = W * H
    idx = np.arange(first_index, first_index + count, dtype=np.int64)
    u = block_uniforms(seed, idx, 0)
    z0, z1 = box_muller(u[0], u[1])
    spx = spread if spread > 0 else W / 20.0
    spy = spread if spread > 0 else H / 20.0
    cx = (W - 1) / 2.0 + z0 * spx
    cy = (H - 1) / 2.0 + z1 * spy
    sx = sigma_lo + (sigma_hi - sigma_lo) * u[2]
    sy = sigma_lo + (sigma_hi - sigma_lo) * u[3] if model == 4 else sx
    alpha = n_signal / (TWO_PI * sx * sy)
    beta = n_background / float(N)
    out = np.empty((count, N), np.float64)
    pix = np.arange(N)
    px = (pix % W).astype(np.float64)
    py = (pix // W).astype(np.float64)
    nblk = (N + 3) // 4
    for lo in range(0, count, 4096):  # bounded temporaries
        hi = min(count, lo + 4096)
        if noise:
            ub = block_uniforms(seed, idx[lo:hi, None], 1 + np.arange(nblk, dtype=np.uint64)[None, :])
            za, zb = box_muller(ub[0], ub[1])
            zc, zd = box_muller(ub[2], ub[3])
            z = np.stack([za, zb, zc, zd], axis=2).reshape(hi - lo, 4 * nblk)[:, :N]
        dx = px[None, :] - cx[lo:hi, None]
        dy = py[None, :] - cy[lo:hi, None]
        sxx, syy = sx[lo:hi, None], sy[lo:hi, None]
        lam = alpha[lo:hi, None] * np.exp(-(dx * dx / (2.0 * sxx * sxx) + dy * dy / (2.0 * syy * syy))) + beta
        v = lam + z * np.sqrt(lam) if noise else lam
        if rounding:
            v = _round_half_away(v)
        if noise and clamp:
            v = np.where(v <= 0.0, 0.0, v)
        out[lo:hi] = v
    cols = [cx, cy, sx] + ([sy] if model == 4 else []) + [alpha, np.full(count, beta)]
    return out, np.stack(cols, axis=1).astype(np.float32)


def simulate_batch(W: int, H: int, count: int, seed: int, model: int = 3, first_index: int = 0,
                   n_signal: float = 400.0, n_background: float = 40.0, sigma_lo: float = 1.0,
                   sigma_hi: float = 2.0, spread: float = 0.0, noise: bool = True, rounding: bool = True):
    """-> images (count, H, W) f32, truth (count, P + 2) f32 [x, y, sigma(s), alpha, beta]."""
    v, truth = _values(W, H, count, seed, model, first_index, n_signal, n_background, sigma_lo, sigma_hi, spread,
                       noise, rounding, clamp=True)
    return v.astype(np.float32).reshape(count, H, W), truth
