"""Every grid W x H with 1 <= W, H <= 32 (all pairwise-tree depths, odd chains, tails, full and masked
geometries): a small batch per grid and model, GPU vs the C oracle bit for bit.
    python tools/geometry_sweep.py [count] [models]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2106_02045_b200 as sf  # noqa: E402
from oracle import initializer as oinit  # noqa: E402
from oracle import lm, oracle_c  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 48
models = [int(m) for m in (sys.argv[2] if len(sys.argv) > 2 else "3,4,5").split(",")]
FIELDS = ("params", "alpha", "beta", "nchi2", "status", "iterations")
bad, n = [], 0
t0 = time.time()
for model in models:
    for W in range(1, 33):
        for H in range(1, 33):
            im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=count, seed=W * 97 + H,
                                                   model=4 if model == 4 else 3))
            im = im.reshape(count, -1)
            ini, amps = oinit.estimate_initial_batch(im, W, H, 0.3, float(max(W, H)), 4 if model == 4 else 3)
            if model == 5:
                ini = np.concatenate([ini, amps], axis=1).astype(np.float32)
            engine = {3: "implicit3", 4: "elliptical", 5: "explicit5"}[model]
            res = sf.fit_batch(im, ini, grid=sf.PixelGrid(W, H), engine=engine)
            ref = oracle_c.fit_batch(im, ini, W, H, lm.LMConfig.for_grid(W, H))
            ok = all(np.array_equal(np.asarray(getattr(res, k)).view(np.uint8), np.asarray(ref[k]).view(np.uint8))
                     for k in FIELDS)
            n += 1
            if not ok:
                bad.append((W, H, model))
print(f"GEOMETRY_SWEEP {n} grids x {count} spots, {len(bad)} mismatching: {bad[:20]} ({time.time() - t0:.0f} s)")
