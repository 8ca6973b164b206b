"""The host pipeline's u16 narrowing of pageable f32 chunks (sf_capi.cu:run_shard, sf_host_narrow.cpp)
never changes a result: batches of several chunks, all-integer or with single non-integer, negative,
-0.0 or > 65535 pixels in some chunks, fit bitwise like the same batch from pinned memory (which is
never narrowed), with and without inits."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("params", "alpha", "beta", "nchi2", "status", "iterations")


@pytest.fixture(scope="module")
def sf():
    import paper_2106_02045_b200 as sf

    sf._lib.require_gpu()
    return sf


def _same(a, b, what):
    for k in FIELDS:
        x, y = np.asarray(getattr(a, k)), np.asarray(getattr(b, k))
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), f"{what}: {k}"


def _pinned_copy(a):
    import torch

    t = torch.from_numpy(a).pin_memory()
    return t


@pytest.mark.parametrize("poison", [None, 0.5, -1.0, -0.0, 70000.0])
def test_pageable_narrowing_is_invisible(sf, poison):
    W = H = 15
    count = 300_000  # several host chunks
    im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=count, seed=314))
    im = im.reshape(count, W * H)
    if poison is not None:
        for s in (5, 150_001, count - 1):  # poison single pixels in the first, a middle and the last chunk
            im[s, 17] = poison
    pinned = _pinned_copy(im)
    ref = sf.fit_batch(pinned, grid=sf.PixelGrid(W, H))  # pinned f32: never narrowed
    got = sf.fit_batch(im, grid=sf.PixelGrid(W, H))      # pageable: narrowed where the chunk allows
    _same(got, ref, f"poison={poison}")
    ini, _ = sf.estimate_initial_batch(im[:20000], 3, grid=sf.PixelGrid(W, H))
    _same(sf.fit_batch(im[:20000], ini, grid=sf.PixelGrid(W, H)),
          sf.fit_batch(_pinned_copy(im[:20000]), ini, grid=sf.PixelGrid(W, H)), "with inits")
