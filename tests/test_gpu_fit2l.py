"""The two-leaves-per-lane kernel (csrc/sf_fit2l.cuh: 4 * SL lanes per spot, profile cache in Tensor
Memory) and the general kernel (sf_fit_kernel.cuh, SPOTFIT_FIT2L=0) give bit-identical fits on every
geometry family the former serves: 2, 4 and 8 leaves, symmetric and elliptical, full and ragged
chains, float and 16-bit pixels.  The selector is read once per process, so each kernel runs in its
own subprocess (SPOTFIT_FIT2L=2 forces the two-leaf kernel below its one-wave threshold)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [(15, 15, 3), (13, 10, 3), (16, 16, 3), (21, 21, 3), (20, 13, 3), (32, 32, 3), (29, 31, 3), (15, 15, 4),
         (21, 21, 4), (24, 24, 4), (32, 30, 4)]

SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2106_02045_b200 as sf
out = {}
for W, H, model in %r:
    im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=3001, seed=W * 100 + H, model=model))
    ini, _ = sf.estimate_initial_batch(im, model, grid=sf.PixelGrid(W, H))
    eng = "elliptical" if model == 4 else "implicit3"
    for u16 in (False, True):
        r = sf.fit_batch(im.astype(np.uint16) if u16 else im, ini, engine=eng, grid=sf.PixelGrid(W, H))
        for k in ("params", "alpha", "beta", "nchi2", "status", "iterations"):
            out["%%d_%%d_%%d_%%d_%%s" %% (W, H, model, u16, k)] = np.asarray(getattr(r, k))
np.savez(sys.argv[1], **out)
''' % (ROOT, CASES)


def run(tmp_path, fit2l):
    path = str(tmp_path / f"fit2l_{fit2l}.npz")
    env = dict(os.environ, SPOTFIT_FIT2L=str(fit2l))
    p = subprocess.run([sys.executable, "-c", SCRIPT, path], env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    return np.load(path)


def test_two_leaf_kernel_equals_general_kernel(tmp_path):
    a, b = run(tmp_path, 2), run(tmp_path, 0)
    assert sorted(a.files) == sorted(b.files)
    bad = [k for k in a.files if not np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8))]
    assert not bad, bad[:10]
