"""Small fits for compute-sanitizer runs (memcheck / racecheck / synccheck): one batch per
geometry family (warp-shared groups, one-leaf groups, one-warp groups, multi-warp groups,
ragged trees, explicit-5), results checked against the C oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2106_02045_b200 as sf  # noqa: E402
from oracle import initializer as oinit  # noqa: E402
from oracle import lm, oracle_c  # noqa: E402

CASES = [(15, 15, 3, 95), (11, 11, 3, 96), (21, 21, 4, 33), (32, 32, 3, 16), (13, 10, 3, 64), (15, 15, 5, 63),
         (1, 5, 3, 65)]
ok = True
for W, H, model, count in CASES:
    im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=count, seed=W * 13 + H, model=min(model, 4)))
    im = im.reshape(count, -1)
    ini, amps = oinit.estimate_initial_batch(im, W, H, 0.3, float(max(W, H)), 4 if model == 4 else 3)
    if model == 5:
        ini = np.concatenate([ini, amps], axis=1).astype(np.float32)
    engine = {3: "implicit3", 4: "elliptical", 5: "explicit5"}[model]
    res = sf.fit_batch(im, ini, grid=sf.PixelGrid(W, H), engine=engine)
    ref = oracle_c.fit_batch(im, ini, W, H, lm.LMConfig.for_grid(W, H))
    same = all(np.array_equal(np.asarray(getattr(res, k)).view(np.uint8), np.asarray(ref[k]).view(np.uint8))
               for k in ("params", "alpha", "beta", "nchi2", "status", "iterations"))
    # the same counts as 16-bit pixels (fit_kernel<..., uint16_t>; odd sizes hit the 2-byte edge copies)
    r16 = sf.fit_batch(im.astype(np.uint16), ini, grid=sf.PixelGrid(W, H), engine=engine)
    same16 = all(np.array_equal(np.asarray(getattr(r16, k)).view(np.uint8), np.asarray(ref[k]).view(np.uint8))
                 for k in ("params", "alpha", "beta", "nchi2", "status", "iterations"))
    ok &= same and same16
    print(f"{W}x{H} P={model}: {'ok' if same else 'MISMATCH'} u16 {'ok' if same16 else 'MISMATCH'}", flush=True)
# the other kernels: GPU initializer, model-level evaluation, device simulator
import torch  # noqa: E402

for W, H in ((15, 15), (21, 21), (32, 32)):
    im, tr = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=40, seed=5))
    ini, _ = sf.estimate_initial_batch(im, 3, grid=sf.PixelGrid(W, H))
    rec = sf.evaluate_batch(im.reshape(40, -1), tr[:, :3], W, H)
    dev = sf.simulate_batch_device(sf.SimConfig(width=W, height=H, count=40, seed=5))
    torch.cuda.synchronize()
# the standalone initializer on every geometry family of its column walk (one column per lane, several
# row segments per column, a 1-row grid, a wide grid with several columns per lane) and on non-integer
# pixels (general path), against the oracle; the fused initializer (inits = None) and the model functions
for W, H in ((15, 15), (5, 9), (1, 7), (9, 1), (40, 1), (13, 10), (32, 32), (11, 11), (21, 21), (16, 3), (13, 13), (9, 2), (15, 3), (17, 5), (25, 3), (27, 27), (20, 30), (20, 20), (18, 7)):
    im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=37, seed=W + 7 * H))
    im = im.reshape(37, -1)
    im[5] += 0.25  # one non-tame spot
    got, _ = sf.estimate_initial_batch(im, 3, grid=sf.PixelGrid(W, H))
    want, _ = oinit.estimate_initial_batch(im, W, H, 0.3, float(max(W, H)), 3)
    same = np.array_equal(got.view(np.uint32), np.asarray(want, np.float32).view(np.uint32))
    ok &= same
    print(f"initializer {W}x{H}: {'ok' if same else 'MISMATCH'}", flush=True)
    sf.fit_batch(im, grid=sf.PixelGrid(W, H))  # fused initializer + fit
    torch.cuda.synchronize()
from paper_2106_02045_b200 import model as sfm  # noqa: E402

g = sfm.SpotImage.from_array(np.float32(np.random.default_rng(1).poisson(20.0, (9, 9))))
shape = sfm.ShapeParams(4.0, 4.0, 1.5)
f, fgrad = sfm.profile_and_gradient(shape, g.grid)
amps, sums = sfm.alpha_beta(f, g)
gs = sfm.gradient_sums(f, fgrad, g, sums)
cg = sfm.coefficient_gradients(sums, gs, amps)
sfm.chi_gradient(g, f, fgrad, amps, cg)
sfm.chi_squared(g, f, amps)
print("SANITIZE_FIT", "ok" if ok else "FAIL")
