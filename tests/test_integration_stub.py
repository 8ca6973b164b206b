"""The ctypes stub of INTEGRATION.md section 1 -- what a maintainer would paste into the reference's
batch engine -- runs as written against this repo's FitConfig / ParameterBounds and the built
library, and returns the batch API's results bitwise."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def stub_source() -> str:
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text.split("## 1.", 1)[1].split("## 2.", 1)[0]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    lib = os.path.join(ROOT, "paper_2106_02045_b200", "_lib", "libspotfit_b200.so")
    assert 'ctypes.CDLL("libspotfit_b200.so")' in code
    return code.replace('ctypes.CDLL("libspotfit_b200.so")', f"ctypes.CDLL({lib!r})")


def test_stub_compiles():
    compile(stub_source(), "INTEGRATION.md", "exec")


@pytest.mark.gpu
def test_stub_matches_fit_batch():
    import paper_2106_02045_b200 as sf

    ns = {}
    exec(compile(stub_source(), "INTEGRATION.md", "exec"), ns)
    W = H = 15
    im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=2000, seed=7))
    ini, _ = sf.estimate_initial_batch(im, 3)
    cfg = sf.FitConfig()
    cfg = sf.FitConfig(bounds=cfg.resolved_bounds(sf.PixelGrid(W, H)))
    out = ns["fit_batch_cuda"](im, ini, cfg, W, H)
    ref = sf.fit_batch(im, ini, config=cfg)
    for k, r in (("params", ref.params), ("alpha", ref.alpha), ("beta", ref.beta), ("nchi2", ref.nchi2),
                 ("status", ref.status), ("iters", ref.iterations)):
        assert np.array_equal(np.asarray(out[k]).view(np.uint8), np.asarray(r).view(np.uint8)), k
