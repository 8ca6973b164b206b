"""Generate the golden fixtures from the REFERENCE itself.

Runs in the build container only (needs /root/reference, which does not
travel to the GPU box).  Imports the reference's own arithmetic
``spotfit.model`` (pkg/src/spotfit/model.py) and records:

  model_golden.npz  per-function outputs of model.py (profile,
                    profile_and_gradient, alpha_beta, chi_squared,
                    gradient_sums, coefficient_gradients, chi_gradient) plus
                    the normal matrix at given (image, params)
                    over several grid shapes, including ragged ones;
  fit_golden.npz    the App. A LM loop (oracle/lm.py:fit_single) driven by the
                    reference model.py on simulated spots + edge cases;
  npexp_golden.npz  np.exp(float32) on hard inputs (the third-party numpy
                    kernel the reference calls at model.py:177,193);
  pwsum_golden.npz  ndarray.sum(dtype=float64) of float32 arrays, n = 1..1024.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from spotfit import model as ref  # noqa: E402  (the reference)

from oracle import initializer, lm  # noqa: E402
from paper_2106_02045_b200.simulator import SimConfig, simulate_batch  # noqa: E402  (input generator only)

SHAPES = [(9, 9), (11, 11), (15, 15), (21, 21), (32, 32), (7, 5), (1, 3), (2, 2), (16, 16), (33, 31), (17, 15),
          (12, 22)]


def model_golden():
    rng = np.random.default_rng(20210604)
    rec = {k: [] for k in ("shape", "image", "params", "singular", "alpha", "beta", "F", "G", "FF", "FG", "denom",
                           "chi", "dF", "dFF", "dFG", "gamma", "dalpha", "dbeta", "grad", "jtj", "f", "fgrad",
                           "f_profile", "has_pixels")}
    for (W, H) in SHAPES:
        N = W * H
        K = 24
        im, tr = simulate_batch(SimConfig(width=W, height=H, count=K, seed=1000 + N))
        for s in range(K):
            g = im[s].reshape(-1).astype(np.float32)
            if s == 0:
                g = np.full(N, 7.0, np.float32)  # constant image
            x, y, sg = tr[s][:3]
            p = [x + rng.normal(0, 0.3), y + rng.normal(0, 0.3), sg * rng.uniform(0.7, 1.4)]
            if s == 1:
                p = [W / 2.0, H / 2.0, 1e4]  # numerically constant profile -> SingularProfile (App. C.4)
            if s == 2:
                p = [0.0, 0.0, 0.3]  # tiny sigma at a corner: denormal / underflowing profile values
            if s == 3:
                p = [W - 1.0, H - 1.0, 0.31]
            sp = ref.ShapeParams(*p)
            grid = ref.PixelGrid(W, H)
            img = ref.SpotImage(grid, g)
            f, fg = ref.profile_and_gradient(sp, grid)
            f2 = ref.profile(sp, grid)
            keep = 1.0 if s < 6 else 0.0  # per-pixel arrays kept for the first cases of each shape only
            row = dict(shape=(W, H), image=np.pad(g, (0, 1024 - N)), params=np.array([sp.x, sp.y, sp.sigma], np.float32),
                       f=np.pad(f * keep, (0, 1024 - N)), fgrad=np.pad(fg * keep, ((0, 1024 - N), (0, 0))),
                       f_profile=np.pad(f2 * keep, (0, 1024 - N)), has_pixels=int(s < 6))
            try:
                amps, sums = ref.alpha_beta(f, img)
                chi = ref.chi_squared(img, f, amps)
                gs = ref.gradient_sums(f, fg, img, sums)
                cg = ref.coefficient_gradients(sums, gs, amps)
                grad, d = ref.chi_gradient(img, f, fg, amps, cg)
                jtj = [float((d[:, j] * d[:, k]).sum(dtype=np.float64)) for j in range(3) for k in range(j, 3)]
                row.update(singular=0, alpha=amps.alpha, beta=amps.beta, F=sums.f_sum, G=sums.g_sum, FF=sums.ff_sum,
                           FG=sums.fg_sum, denom=sums.denom, chi=chi, dF=gs.df, dFF=gs.dff, dFG=gs.dfg,
                           gamma=gs.gamma, dalpha=cg[0], dbeta=cg[1], grad=grad, jtj=jtj)
            except ref.SingularProfile:
                z3 = np.zeros(3)
                row.update(singular=1, alpha=np.nan, beta=np.nan, F=np.nan, G=np.nan, FF=np.nan, FG=np.nan,
                           denom=np.nan, chi=np.nan, dF=z3, dFF=z3, dFG=z3, gamma=z3, dalpha=z3, dbeta=z3, grad=z3,
                           jtj=np.zeros(6))
            for k, v in row.items():
                rec[k].append(v)
    out = {}
    for k, v in rec.items():
        a = np.array(v)
        if k in ("alpha", "beta", "chi"):
            a = a.astype(np.float32)
        out[k] = a
    np.savez_compressed(os.path.join(HERE, "model_golden.npz"), **out)
    print("model_golden:", len(rec["alpha"]), "cases")


FIT_SETS = [((11, 11), 300, 11), ((15, 15), 300, 15), ((21, 21), 80, 21), ((32, 32), 40, 32), ((9, 9), 120, 9),
            ((7, 5), 40, 75), ((17, 15), 40, 1715)]


def fit_golden():
    out = {}
    for (W, H), K, seed in FIT_SETS:
        N = W * H
        im, tr = simulate_batch(SimConfig(width=W, height=H, count=K, seed=seed,
                                          n_signal=1600.0 if seed == 9 else 400.0))
        im = im.reshape(K, N)
        cfg = lm.LMConfig.for_grid(W, H)
        inits, _ = initializer.estimate_initial_batch(im, W, H, cfg.sigma_min, cfg.sigma_max)
        if seed == 15:
            # edge cases on the headline grid
            im[0] = 7.0  # constant image
            nl, ntr = simulate_batch(SimConfig(width=W, height=H, count=1, seed=99, noise=False, rounding=False))
            im[1] = nl.reshape(-1)  # noiseless, unrounded: exact recovery expected
            inits[1] = initializer.estimate_initial(nl[0], cfg.sigma_min, cfg.sigma_max)[0]
            im[2, 5] = np.nan  # InvalidInput
            inits[3] = [-50.0, 80.0, 100.0]  # init far out of bounds -> limit()
            inits[4] = [7.0, 7.0, np.inf]  # non-finite init -> InvalidInput
            im[5] = 0.0
            im[5, 112] = 1000.0  # single hot pixel
        res = lm.fit_batch_arrays(ref, im, inits, W, H, cfg)
        key = f"{W}x{H}"
        out[f"{key}_images"] = im.astype(np.float32)
        out[f"{key}_inits"] = inits.astype(np.float32)
        for k, v in res.items():
            out[f"{key}_{k}"] = v
        print("fit_golden", key, K, "mean it", res["iterations"].mean(), "stops", np.bincount(res["status"] & 7, minlength=5))
    # the damped solve (SPEC.md:195-196 examples + random SPD)
    rng = np.random.default_rng(5)
    jt, rh, la, de, ok = [], [], [], [], []
    for t in range(200):
        if t == 0:
            J, r, lam = np.eye(3), np.array([1.0, 2.0, 3.0]), 0.0
        elif t == 1:
            J, r, lam = np.eye(3), np.array([1.0, 2.0, 3.0]), 1.0
        elif t == 2:
            J, r, lam = np.zeros((3, 3)), np.zeros(3), 0.01
        else:
            A = rng.normal(size=(3, 3)) * 10 ** rng.uniform(-3, 3)
            J, r, lam = A @ A.T, rng.normal(size=3), 10.0 ** rng.integers(-6, 4)
        packed = [J[i, j] for i in range(3) for j in range(i, 3)]
        d = lm.solve_step(packed, r, lam)
        jt.append(packed), rh.append(r), la.append(lam), ok.append(d is not None)
        de.append(d if d is not None else [np.nan] * 3)
    out["solve_jtj"], out["solve_rhs"], out["solve_lam"] = np.array(jt), np.array(rh), np.array(la)
    out["solve_delta"], out["solve_ok"] = np.array(de), np.array(ok)
    np.savez_compressed(os.path.join(HERE, "fit_golden.npz"), **out)


def npexp_golden():
    rng = np.random.default_rng(3)
    hard = [0.0, -0.0, -1e-45, -1e-38, -0.5, -1.0, -87.0, -87.3, -88.0, -100.0, -103.0, -103.97207641601562,
            -103.97208404541015625, -103.9721, -104.0, -200.0, -np.inf, np.nan]
    x = np.concatenate([np.array(hard, np.float32), -rng.uniform(0, 104, 20000).astype(np.float32),
                        -(10.0 ** rng.uniform(-40, 2, 5000)).astype(np.float32)])
    with np.errstate(all="ignore"):
        np.savez_compressed(os.path.join(HERE, "npexp_golden.npz"), x=x, y=np.exp(x))


def pwsum_golden():
    rng = np.random.default_rng(4)
    xs, sums = [], []
    ns = list(range(1, 300)) + list(range(300, 1025, 7)) + [1023, 1024]
    for n in ns:
        x = (rng.standard_normal(n) * 10.0 ** rng.uniform(-6, 6, n)).astype(np.float32)
        xs.append(np.pad(x, (0, 1024 - n)))
        sums.append(x.sum(dtype=np.float64))
    np.savez_compressed(os.path.join(HERE, "pwsum_golden.npz"), x=np.array(xs), s=np.array(sums), n=np.array(ns))


def model_pixels_golden():
    """Per-pixel outputs of every spotfit.model function (h, r, dmat besides f, fgrad), also on
    profile / gradient arrays that did not come from profile_and_gradient (uniform random f in
    [0, 1), normal fgrad): the GPU's sf_model_* entry points are checked against these."""
    rng = np.random.default_rng(20260101)
    rec = {k: [] for k in ("shape", "image", "params", "f", "fgrad", "f_profile", "kind", "singular", "alpha", "beta",
                           "sums", "h", "r", "chi", "gsums", "dalpha", "dbeta", "grad", "dmat")}
    for (W, H) in SHAPES:
        N = W * H
        im, tr = simulate_batch(SimConfig(width=W, height=H, count=4, seed=5000 + N))
        for s in range(4):
            g = im[s].reshape(-1).astype(np.float32)
            x, y, sg = tr[s][:3]
            sp = ref.ShapeParams(x + rng.normal(0, 0.3), y + rng.normal(0, 0.3), sg * rng.uniform(0.7, 1.4))
            grid = ref.PixelGrid(W, H)
            img = ref.SpotImage(grid, g)
            f_prof = ref.profile(sp, grid)
            if s < 2:  # the reference chain as the solver runs it
                f, fg = ref.profile_and_gradient(sp, grid)
                kind = 0
            else:  # arbitrary arrays through the same functions
                f = rng.uniform(0.0, 1.0, N).astype(np.float32)
                fg = rng.normal(0.0, 1.0, (N, 3)).astype(np.float32)
                kind = 1
            if s == 3:
                f = np.full(N, 0.25, np.float32)  # constant profile: SingularProfile
            row = dict(shape=(W, H), image=np.pad(g, (0, 1024 - N)),
                       params=np.array([sp.x, sp.y, sp.sigma], np.float32), f=np.pad(f, (0, 1024 - N)),
                       fgrad=np.pad(fg, ((0, 1024 - N), (0, 0))), f_profile=np.pad(f_prof, (0, 1024 - N)), kind=kind)
            try:
                amps, sums = ref.alpha_beta(f, img)
                h = ref.model_values(f, amps)
                r = ref.residuals(img, f, amps)
                chi = ref.chi_squared(img, f, amps)
                gs = ref.gradient_sums(f, fg, img, sums)
                cg = ref.coefficient_gradients(sums, gs, amps)
                grad, d = ref.chi_gradient(img, f, fg, amps, cg)
                row.update(singular=0, alpha=amps.alpha, beta=amps.beta,
                           sums=[sums.f_sum, sums.g_sum, sums.ff_sum, sums.fg_sum, sums.denom],
                           h=np.pad(h, (0, 1024 - N)), r=np.pad(r, (0, 1024 - N)), chi=chi,
                           gsums=np.stack([gs.df, gs.dff, gs.dfg, gs.gamma]), dalpha=cg[0], dbeta=cg[1], grad=grad,
                           dmat=np.pad(d, ((0, 1024 - N), (0, 0))))
            except ref.SingularProfile:
                nan = np.float32(np.nan)
                row.update(singular=1, alpha=nan, beta=nan, sums=[np.nan] * 5, h=np.zeros(1024, np.float32),
                           r=np.zeros(1024, np.float32), chi=nan, gsums=np.zeros((4, 3)), dalpha=np.zeros(3),
                           dbeta=np.zeros(3), grad=np.zeros(3), dmat=np.zeros((1024, 3), np.float32))
            for k, v in row.items():
                rec[k].append(v)
    out = {}
    for k, v in rec.items():
        a = np.array(v)
        if k in ("alpha", "beta", "chi", "f", "fgrad", "f_profile", "h", "r", "dmat", "image", "params"):
            a = a.astype(np.float32)
        out[k] = a
    np.savez_compressed(os.path.join(HERE, "model_pixels_golden.npz"), **out)
    print("model_pixels_golden:", len(rec["alpha"]), "cases")


if __name__ == "__main__":
    import sys as _sys

    which = _sys.argv[1:] or ["model", "fit", "npexp", "pwsum", "model_pixels"]
    for name in which:
        globals()[f"{name}_golden"]()
