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


@pytest.mark.parametrize("W,H,model,kw", [(15, 15, 3, {}), (21, 21, 4, {}), (11, 11, 3, {"first_index": 10**9}),
                                           (32, 32, 3, {"spread": 2.5}), (7, 5, 4, {"noise": False}),
                                           (9, 9, 3, {"noise": False, "rounding": False}),
                                           (13, 3, 3, {"n_signal": 4000.0, "n_background": 400.0})])
def test_numpy_restatement_equals_host_generator(W, H, model, kw):
    """oracle/simulator.py (vectorised numpy Philox + Box-Muller + SPEC.md:335-358 noise) equals
    the product's host generator bit for bit on every pixel and truth value."""
    import paper_2106_02045_b200 as sf
    from oracle import simulator as osim

    first = kw.pop("first_index", 0)
    count = 3000
    a, ta = osim.simulate_batch(W, H, count, seed=0xDEADBEEF12345, model=model, first_index=first, **kw)
    ckw = {("center_spread" if k == "spread" else k): v for k, v in kw.items()}
    b, tb = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=count, seed=0xDEADBEEF12345, model=model, **ckw),
                              first_index=first)
    assert bits_equal(a, b) and bits_equal(ta, tb)


@pytest.mark.gpu
def test_device_simulator_matches_independent_restatement():
    """Every pixel of sampled spots of the DEVICE generator against the independent numpy
    restatement (oracle/simulator.py): equal except where the unrounded value lies within
    1e-6 of a .5 rounding boundary (CUDA's f64 libm and numpy's may differ in the last ulp)."""
    import torch

    import paper_2106_02045_b200 as sf
    from oracle import simulator as osim

    for model, W, count in ((3, 15, 200_000), (4, 21, 50_000), (3, 32, 20_000)):
        cfg = sf.SimConfig(width=W, height=W, count=count, seed=2021, model=model)
        di, dt = sf.simulate_batch_device(cfg)
        torch.cuda.synchronize()
        idx = np.unique(np.linspace(0, count - 1, 1500).astype(np.int64))
        di, dt = di.cpu().numpy()[idx].reshape(len(idx), -1), dt.cpu().numpy()[idx]
        oi = np.concatenate([osim.simulate_batch(W, W, 1, 2021, model, first_index=int(i))[0].reshape(1, -1)
                             for i in idx])
        ot = np.concatenate([osim.simulate_batch(W, W, 1, 2021, model, first_index=int(i))[1] for i in idx])
        rows, cols = np.nonzero(di != oi)
        for r, c in zip(rows, cols):
            v = osim.unrounded(W, W, int(idx[r]), 2021, model)[c]
            assert abs(abs(v - np.trunc(v)) - 0.5) < 1e-6 and abs(di[r, c] - oi[r, c]) == 1, (model, idx[r], c, v)
        rel = np.abs(dt.astype(np.float64) - ot) / np.maximum(np.abs(ot), 1e-30)
        assert rel.max() < 1e-6 and (dt == ot).mean() > 0.999


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
