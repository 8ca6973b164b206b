"""The host pipeline's u16 narrowing of f32 chunks (sf_capi.cu:run_shard, sf_host_narrow.cpp), for
pageable and pinned input, never changes a result: batches of several chunks, all-integer or with
single non-integer, negative, -0.0 or > 65535 pixels in some chunks, fit bitwise like the same batch
resident on the device (no host pipeline), with and without inits.  The first chunk that does not
narrow ends narrowing for the rest of the call; pinned input narrows a share of its chunks
(sf_stats.n_chunks_u16, sf_stats.h2d_bytes)."""
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
@pytest.mark.parametrize("where", ["first", "middle"])
def test_narrowing_is_invisible(sf, poison, where):
    import torch

    W = H = 15
    count = 300_000  # several host chunks
    if poison is None and where == "middle":
        pytest.skip("same as first")
    im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=count, seed=314))
    im = im.reshape(count, W * H)
    if poison is not None:
        spots = (5, 150_001, count - 1) if where == "first" else (150_001,)
        for s in spots:
            im[s, 17] = poison
    grid = sf.PixelGrid(W, H)
    ref = sf.fit_batch(torch.from_numpy(im).cuda(), grid=grid)  # device-resident: no host pipeline
    for label, src in (("pageable", im), ("pinned", _pinned_copy(im).numpy())):
        got = sf.fit_batch(src, grid=grid)
        _same(got, ref, f"{label} poison={poison} {where}")
        n, n16, nb = got.stats["n_chunks"], got.stats["n_chunks_u16"], got.stats["h2d_bytes"]
        assert count * W * H * 2 <= nb <= count * W * H * 4, (label, got.stats)
        if label == "pinned":  # a share of the chunks (never the first; only while the host keeps up)
            assert n16 < n, (label, got.stats)
        elif poison is None:
            assert n16 == n and nb == count * W * H * 2, (label, got.stats)
        elif where == "first":
            assert n16 == 0, (label, got.stats)
        else:
            assert 0 < n16 < n, (label, got.stats)  # narrowed up to the poisoned chunk, f32 from there on
    ini, _ = sf.estimate_initial_batch(im[:20000], 3, grid=grid)
    ref_i = sf.fit_batch(torch.from_numpy(im[:20000]).cuda(), torch.from_numpy(ini).cuda(), grid=grid)
    _same(sf.fit_batch(im[:20000], ini, grid=grid), ref_i, "pageable with inits")
    _same(sf.fit_batch(_pinned_copy(im[:20000]).numpy(), _pinned_copy(ini).numpy(), grid=grid), ref_i,
          "pinned with inits")
