"""Pins the third-party numeric substrate the reference stands on:
numpy's float32 exp (model.py:177,193) and float64 pairwise sum
(model.py:222-225,250,263-265,314), against the committed fixtures made by the
reference's own numpy and against this host's live numpy."""
import numpy as np
import pytest

from conftest import bits_equal, load_golden


def test_npexp_matches_golden(oracle_lib):
    d = load_golden("npexp_golden.npz")
    assert bits_equal(oracle_lib.npexp(d["x"]), d["y"])


def test_npexp_matches_live_numpy_sample(oracle_lib):
    # self-check that this host's numpy dispatches the same exp kernel (App. B.2)
    rng = np.random.default_rng(11)
    x = np.concatenate([-rng.uniform(0, 104, 2_000_000), -(10.0 ** rng.uniform(-45, 2.02, 200_000))]).astype(np.float32)
    assert bits_equal(oracle_lib.npexp(x), np.exp(x))


@pytest.mark.slow
def test_npexp_exhaustive_negative_range(oracle_lib):
    """All 1,120,927,745 float32 in [-104, -0] -- ~1 min."""
    lo = int(np.float32(-104.0).view(np.uint32))
    u = 0x80000000
    while u <= lo:
        hi = min(u + (1 << 24), lo + 1)
        x = np.arange(u, hi, dtype=np.uint64).astype(np.uint32).view(np.float32)
        assert bits_equal(oracle_lib.npexp(x), np.exp(x))
        u = hi


def test_pairwise_sum_matches_golden(oracle_lib):
    d = load_golden("pwsum_golden.npz")
    for row, n, ref in zip(d["x"], d["n"], d["s"]):
        assert oracle_lib.pw_sum(row[:n]) == ref


def test_pairwise_sum_matches_live_numpy(oracle_lib):
    rng = np.random.default_rng(12)
    for n in list(range(1, 260)) + [441, 511, 512, 513, 1000, 1023, 1024]:
        x = (rng.standard_normal(n) * 10.0 ** rng.uniform(-4, 4, n)).astype(np.float32)
        assert oracle_lib.pw_sum(x) == x.sum(dtype=np.float64)


def test_exp_underflow_clamp_equals_guard():
    """The kernel's packed exp replaces numpy's underflow guard (x <= -103.97208 -> +0) by
    clamping x at -104 (sf_device.cuh:npexp2).  Equal bit for bit on every float32 in
    [-200, -100] (the guard region and far below it) and on the clamp value itself."""
    from oracle import oracle_c

    lib = oracle_c.lib()
    assert lib.npexp_clamp_mismatches(-200.0, -100.0) == 0
    for x in (-1e30, -3.4e38, -104.0, -103.97208404541015625):
        assert lib.npexp_f32_clamped(x) == 0.0 and lib.npexp_f32(x) == 0.0
