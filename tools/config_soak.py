"""Randomised parity soak over the configuration space: grid (1..32 x 1..32), model (3 / 4 / 5),
every FitConfig knob (iteration budget, max_error, min_delta, min_step, lambda schedule),
ParameterBounds (margins, sigma range) and simulator settings (signal, background, sigma
range, centre spread, noise on/off), with perturbed initial guesses.  Each round fits a
batch on the GPU and compares every result field bitwise with the C oracle.

    python tools/config_soak.py [rounds] [seed]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2106_02045_b200 as sf  # noqa: E402
from oracle import initializer as oinit  # noqa: E402
from oracle import lm, oracle_c  # noqa: E402

FIELDS = ("params", "alpha", "beta", "nchi2", "status", "iterations")


def log_uniform(rng, lo, hi):
    return float(10.0 ** rng.uniform(np.log10(lo), np.log10(hi)))


def make_case(rng, models=(3, 3, 4, 5), counts=(200, 3000)):
    """One random case: grid, model, FitConfig kwargs + bounds (GPU and oracle forms), images, inits."""
    W, H = int(rng.integers(1, 33)), int(rng.integers(1, 33))
    model = int(rng.choice(list(models)))
    count = int(rng.integers(*counts))
    S = max(W, H)
    smin = float(rng.uniform(0.1, 0.8))
    kw = dict(max_iterations=int(rng.integers(1, 41)),
              max_error=0.0 if rng.random() < 0.7 else log_uniform(rng, 1.0, 1e4),
              min_delta=log_uniform(rng, 1e-9, 1e-2), min_step=log_uniform(rng, 1e-7, 1e-2),
              lambda_init=log_uniform(rng, 1e-4, 1.0), lambda_up=float(rng.uniform(1.5, 20.0)),
              lambda_down=float(rng.uniform(1.5, 20.0)))
    kw["lambda_max"] = kw["lambda_init"] * log_uniform(rng, 10.0, 1e8)
    mx, my = float(rng.uniform(0.0, W)), float(rng.uniform(0.0, H))
    smax = float(rng.uniform(smin + 0.5, 2.0 * S + 1.0))
    bounds = sf.ParameterBounds(mx, my, smin, smax)
    cfg = sf.FitConfig(bounds=bounds, **kw)
    ocfg = lm.LMConfig(margin_x=mx, margin_y=my, sigma_min=smin, sigma_max=smax, **kw)
    lo_s = float(rng.uniform(0.5, 2.0))
    sim = sf.SimConfig(width=W, height=H, count=count, seed=int(rng.integers(1 << 30)), model=min(model, 4),
                       n_signal=log_uniform(rng, 20.0, 2e5), n_background=float(rng.choice([0.0, 5.0, 40.0, 400.0])),
                       sigma_range=(lo_s, lo_s + float(rng.uniform(0.0, 2.0))),
                       center_spread=float(rng.choice([0.0, 0.5, 2.0])), noise=bool(rng.random() < 0.85))
    im, _ = sf.simulate_batch(sim)
    im = im.reshape(count, -1)
    if rng.random() < 0.2:  # background-subtracted data: negative pixels
        im = (im - np.float32(rng.uniform(0.0, 50.0))).astype(np.float32)
    ini, amps = oinit.estimate_initial_batch(im, W, H, smin, smax, 4 if model == 4 else 3)
    ini = ini + rng.normal(0.0, 0.3, ini.shape).astype(np.float32) * (rng.random() < 0.5)
    if model == 5:
        ini = np.concatenate([ini, amps], axis=1)
    ini = np.ascontiguousarray(ini, dtype=np.float32)
    return dict(W=W, H=H, model=model, count=count, kw=kw, cfg=cfg, ocfg=ocfg, im=im, ini=ini)


def one_round(rng, r):
    c = make_case(rng)
    W, H, model, count, kw, cfg, ocfg, im, ini = (c[k] for k in ("W", "H", "model", "count", "kw", "cfg", "ocfg",
                                                                 "im", "ini"))
    engine = {3: "implicit3", 4: "elliptical", 5: "explicit5"}[model]
    res = sf.fit_batch(im, ini, config=cfg, grid=sf.PixelGrid(W, H), engine=engine)
    ref = oracle_c.fit_batch(im, ini, W, H, ocfg)
    bad = [k for k in FIELDS if not np.array_equal(np.asarray(getattr(res, k)).view(np.uint8),
                                                   np.asarray(ref[k]).view(np.uint8))]
    if np.all(im >= 0) and np.all(im < 65536) and np.array_equal(im, np.round(im)):  # camera counts: u16 path too
        r16 = sf.fit_batch(im.astype(np.uint16), ini, config=cfg, grid=sf.PixelGrid(W, H), engine=engine)
        bad += [k + "(u16)" for k in FIELDS if not np.array_equal(np.asarray(getattr(r16, k)).view(np.uint8),
                                                                 np.asarray(ref[k]).view(np.uint8))]
    stops = np.bincount(np.asarray(res.status) & 7, minlength=5)
    print(f"round {r:4d}: {W:2d}x{H:2d} P={model} n={count:4d} it<={kw['max_iterations']:2d} "
          f"stops={stops.tolist()} {'ok' if not bad else 'MISMATCH ' + ','.join(bad)}", flush=True)
    return count, not bad


if __name__ == "__main__":
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2106)
    t0, fits, fails = time.time(), 0, 0
    for r in range(rounds):
        n, ok = one_round(rng, r)
        fits += n
        fails += not ok
    print(f"CONFIG_SOAK rounds={rounds} fits={fits} mismatching_rounds={fails} ({time.time() - t0:.0f} s)")
