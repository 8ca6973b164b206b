"""Simulator: counter-based determinism, index
regeneration, the paper's distribution parameters, and a
pure-Python restatement of the Philox stream."""
import math

import numpy as np
import pytest

from conftest import bits_equal


def _sim(**kw):
    import paper_2106_02045_b200 as sf

    return sf.simulate_batch(sf.SimConfig(**kw))


def test_deterministic_and_index_regeneration():
    import paper_2106_02045_b200 as sf

    cfg = sf.SimConfig(width=15, height=15, count=300, seed=7)
    a, ta = sf.simulate_batch(cfg)
    b, tb = sf.simulate_batch(cfg, threads=1)
    assert bits_equal(a, b) and bits_equal(ta, tb)  # thread count does not matter
    for idx in (0, 1, 123, 299):
        im, tr = sf.simulate_spot(cfg, idx)
        assert bits_equal(im, a[idx]) and bits_equal(tr, ta[idx])
    c, _ = sf.simulate_batch(sf.SimConfig(width=15, height=15, count=300, seed=8))
    assert not np.array_equal(a, c)


def test_distribution_parameters():
    S = 9
    im, tr = _sim(width=S, height=S, count=100_000, seed=3)
    cx, cy, sg = tr[:, 0], tr[:, 1], tr[:, 2]
    for c in (cx, cy):  # centre ~ N((S-1)/2, S/20)
        assert abs(c.mean() - (S - 1) / 2) < 0.01
        assert abs(c.std() / (S / 20) - 1) < 0.03
    assert sg.min() >= 1.0 and sg.max() <= 2.0 and abs(sg.mean() - 1.5) < 0.01
    assert np.allclose(tr[:, 3], 400.0 / (2 * np.pi * tr[:, 2].astype(np.float64) ** 2), rtol=1e-5)
    assert np.all(tr[:, 4] == np.float32(40.0 / 81))
    assert np.all(im >= 0) and np.all(im == np.round(im))  # non-negative integers


def test_noise_disabled_cases():
    im, _ = _sim(width=9, height=9, count=20, seed=1, n_signal=0.0, noise=False)
    assert np.all(im == round(40.0 / 81))
    im, tr = _sim(width=9, height=9, count=50, seed=1, noise=False, rounding=False)
    # unrounded noiseless: alpha*f + beta exactly (f64 then f32)
    x, y = np.meshgrid(np.arange(9), np.arange(9))
    for s in range(5):
        cx, cy, sg, a, b = (float(v) for v in tr[s])
        assert np.allclose(im[s], a * np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2 * sg * sg)) + b, rtol=1e-5)


def _philox(c, k0, k1):
    M = 0xFFFFFFFF
    c = list(c)
    for _ in range(10):
        p0 = 0xD2511F53 * c[0]
        p1 = 0xCD9E8D57 * c[2]
        c = [((p1 >> 32) ^ c[1] ^ k0) & M, p1 & M, ((p0 >> 32) ^ c[3] ^ k1) & M, p0 & M]
        k0 = (k0 + 0x9E3779B9) & M
        k1 = (k1 + 0xBB67AE85) & M
    return c


def test_python_restatement_of_the_stream():
    """Philox4x32-10 + Box-Muller restated in Python reproduces the C truth draws."""
    seed, W = 0x1234567890ABCDEF, 11
    _, tr = _sim(width=W, height=W, count=8, seed=seed)
    for idx in range(8):
        c = _philox([idx & 0xFFFFFFFF, idx >> 32, 0, 0x53504F54], seed & 0xFFFFFFFF, seed >> 32)
        u = [(v + 0.5) * 2.3283064365386963e-10 for v in c]
        r = math.sqrt(-2.0 * math.log(u[0]))
        cx = (W - 1) / 2.0 + r * math.cos(6.283185307179586 * u[1]) * (W / 20.0)
        sg = 1.0 + 1.0 * u[2]
        assert np.float32(cx) == tr[idx, 0] and np.float32(sg) == tr[idx, 2]


@pytest.mark.gpu
def test_device_simulator_matches_host():
    import torch

    import paper_2106_02045_b200 as sf

    for model, W in ((3, 15), (4, 21), (3, 32)):
        cfg = sf.SimConfig(width=W, height=W, count=50_000, seed=99, model=model)
        hi, ht = sf.simulate_batch(cfg)
        di, dt = sf.simulate_batch_device(cfg)
        torch.cuda.synchronize()
        di, dt = di.cpu().numpy(), dt.cpu().numpy()
        diff = di != hi
        assert diff.mean() < 1e-6 and (np.abs(di - hi)[diff] <= 1).all()  # .5-boundary libm ulp only
        rel = np.abs(dt.astype(np.float64) - ht) / np.maximum(np.abs(ht), 1e-30)
        assert rel.max() < 1e-6 and (dt == ht).mean() > 0.999
