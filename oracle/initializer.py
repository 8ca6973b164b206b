"""Restated SPEC initializer (TEST INFRASTRUCTURE ONLY).

SPEC.md:276-305 (smooth3x3, estimate_initial), with the
arithmetic pinned exactly as csrc/sf_init.cu computes it:
  smoothed_i = f32(sum_f64(in-bounds 3x3 neighbours, row-major) / count)
  centre = first maximum of smoothed (row-major); beta = min smoothed;
  alpha = f32(f64(max) - f64(beta)); M = #{g_i > alpha*exp(-0.5) + beta} (f64)
  sigma = f32(clamp(sqrt(M/pi), sigma_min, sigma_max)).
"""
from __future__ import annotations

import math

import numpy as np

EXP_MINUS_HALF = float.fromhex("0x1.368b2fc6f960ap-1")


def smooth3x3(img2d: np.ndarray) -> np.ndarray:
    """truncated-window mean."""
    H, W = img2d.shape
    out = np.empty((H, W), np.float32)
    for y in range(H):
        for x in range(W):
            s, c = 0.0, 0
            for dy in (-1, 0, 1):
                yy = y + dy
                if not 0 <= yy < H:
                    continue
                for dx in (-1, 0, 1):
                    xx = x + dx
                    if 0 <= xx < W:
                        s += float(img2d[yy, xx])
                        c += 1
            out[y, x] = np.float32(s / c)
    return out


def estimate_initial(img2d: np.ndarray, sigma_min: float, sigma_max: float, model: int = 3):
    """SPEC.md:286-290 -> (params[model] f32, alpha f32, beta f32)."""
    H, W = img2d.shape
    sm = smooth3x3(np.asarray(img2d, np.float32)).reshape(-1)
    best, idx = sm[0], 0
    for i in range(1, sm.size):
        if sm[i] > best:
            best, idx = sm[i], i
    lo = float(sm.min())
    alpha = float(np.float32(float(best) - lo))
    thr = alpha * EXP_MINUS_HALF + lo
    M = int(np.sum(np.asarray(img2d, np.float64).reshape(-1) > thr))
    sg = math.sqrt(M / math.pi)
    sg = sigma_min if sg < sigma_min else (sigma_max if sg > sigma_max else sg)
    p = [float(idx % W), float(idx // W), float(np.float32(sg))]
    if model == 4:
        p.append(p[2])
    return np.array(p, np.float32), np.float32(alpha), np.float32(lo)


def estimate_initial_batch(images: np.ndarray, W: int, H: int, sigma_min: float, sigma_max: float, model: int = 3):
    count = images.shape[0]
    out = np.empty((count, model), np.float32)
    amps = np.empty((count, 2), np.float32)
    for s in range(count):
        p, a, b = estimate_initial(images[s].reshape(H, W), sigma_min, sigma_max, model)
        out[s], amps[s] = p, (a, b)
    return out, amps


def estimate_initial_batch_np(images: np.ndarray, W: int, H: int, sigma_min: float, sigma_max: float,
                              model: int = 3):
    """estimate_initial_batch vectorised over spots (same results, bit for bit): the 3x3 sums run
    over a zero-padded f64 copy in the same row-major neighbour order (a +0.0 pad leaves every
    partial sum unchanged, since a sum starting at +0.0 is never -0.0).  Rows holding a
    non-finite pixel go through the scalar loop (numpy's argmax treats NaN differently from the
    strict ">" scan)."""
    count = images.shape[0]
    g = np.asarray(images, np.float32).reshape(count, H, W)
    pad = np.zeros((count, H + 2, W + 2), np.float64)
    pad[:, 1:-1, 1:-1] = g
    s = np.zeros((count, H, W), np.float64)
    for dy in range(3):
        for dx in range(3):
            s = s + pad[:, dy:dy + H, dx:dx + W]
    cy = 1 + (np.arange(H) > 0) + (np.arange(H) < H - 1)
    cx = 1 + (np.arange(W) > 0) + (np.arange(W) < W - 1)
    sm = (s / (cy[:, None] * cx[None, :]).astype(np.float64)).astype(np.float32).reshape(count, -1)
    idx = np.argmax(sm, axis=1)  # first maximum (finite rows)
    best = sm[np.arange(count), idx].astype(np.float64)
    lo = sm.min(axis=1).astype(np.float64)
    alpha = (best - lo).astype(np.float32)
    thr = alpha.astype(np.float64) * EXP_MINUS_HALF + lo
    M = np.sum(g.reshape(count, -1).astype(np.float64) > thr[:, None], axis=1)
    sg = np.sqrt(M / math.pi)
    sg = np.where(sg < sigma_min, sigma_min, np.where(sg > sigma_max, sigma_max, sg)).astype(np.float32)
    out = np.empty((count, model), np.float32)
    out[:, 0] = (idx % W).astype(np.float32)
    out[:, 1] = (idx // W).astype(np.float32)
    out[:, 2] = sg
    if model == 4:
        out[:, 3] = sg
    amps = np.stack([alpha, lo.astype(np.float32)], axis=1)
    bad = ~np.all(np.isfinite(g.reshape(count, -1)), axis=1)
    for r in np.nonzero(bad)[0]:
        p, a, b = estimate_initial(g[r], sigma_min, sigma_max, model)
        out[r], amps[r] = p, (a, b)
    return out, amps
