"""Fused initializer (inits=None -> sf_fit_kernel.cuh:fused_init), the standalone
initializer on non-finite images, and the C-ABI's argument / device / work-slot
guards.  Run on a B200: pytest -m gpu."""
import ctypes

import numpy as np
import pytest

from conftest import bits_equal
from oracle import initializer as oinit
from oracle import lm

pytestmark = pytest.mark.gpu

FIELDS = ("params", "alpha", "beta", "nchi2", "status", "iterations")


@pytest.fixture(scope="module")
def sf():
    import paper_2106_02045_b200 as sf

    sf._lib.require_gpu()
    return sf


def _sim(sf, W, H, count, seed, model=3):
    im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=count, seed=seed, model=model))
    return im.reshape(count, -1)


def _same(a, b, label):
    for k in FIELDS:
        x, y = np.asarray(getattr(a, k)), np.asarray(b[k] if isinstance(b, dict) else getattr(b, k))
        assert bits_equal(x, y), f"{label}: field {k} differs ({np.mean(x != y):.3g} of entries)"


def _standalone_inits(sf, im, W, H, P):
    model = 3 if P == 5 else P
    ini, amps = sf.estimate_initial_batch(im, model, grid=sf.PixelGrid(W, H))
    if P == 5:  # explicit-5 starts from (x, y, sigma, alpha, beta) of the initializer
        ini = np.ascontiguousarray(np.concatenate([ini, amps], axis=1).astype(np.float32))
    return ini


# every geometry family: 1/2/4/8(2-warp CTA)/16(4-warp CTA) slots, ragged and full chains
GRIDS = [(15, 15, "implicit3"), (11, 11, "implicit3"), (21, 21, "elliptical"), (32, 32, "implicit3"),
         (31, 33, "implicit3"), (7, 5, "implicit3"), (1, 1, "implicit3"), (1, 1024, "implicit3"),
         (13, 11, "explicit5"), (32, 32, "elliptical"), (24, 21, "elliptical")]


@pytest.mark.parametrize("W,H,engine", GRIDS)
def test_fused_init_equals_standalone_initializer(sf, W, H, engine):
    """fit_batch(images) estimates the inits inside the fit kernel from the staged spot:
    bitwise the fits of fit_batch(images, standalone_inits), on host f32 / u16 and
    device f32 / u16 inputs."""
    import torch

    P = sf.batch_engine.ENGINES[engine]
    count = 6001 if W * H <= 256 else 2501
    im = _sim(sf, W, H, count, seed=90 + W * 7 + H, model=4 if P == 4 else 3)
    grid = sf.PixelGrid(W, H)
    ref = sf.fit_batch(im, _standalone_inits(sf, im, W, H, P), grid=grid, engine=engine)
    _same(sf.fit_batch(im, grid=grid, engine=engine), ref, f"host f32 {W}x{H} {engine}")
    u = im.astype(np.uint16)
    assert np.array_equal(u.astype(np.float32), im)
    _same(sf.fit_batch(u, grid=grid, engine=engine), ref, f"host u16 {W}x{H} {engine}")
    _same(sf.fit_batch(torch.from_numpy(im).cuda(), grid=grid, engine=engine), ref, f"device f32 {W}x{H} {engine}")
    _same(sf.fit_batch(torch.from_numpy(u).cuda(), grid=grid, engine=engine), ref, f"device u16 {W}x{H} {engine}")


@pytest.mark.parametrize("W,H,engine", [(15, 15, "implicit3"), (11, 11, "implicit3"), (21, 21, "elliptical"),
                                        (32, 32, "implicit3"), (13, 11, "explicit5"), (5, 40, "implicit3"),
                                        (1, 200, "implicit3")])
def test_inits_none_large_batches(sf, W, H, engine):
    """Batches above the fused-initializer size (sf_launch.h:kFusedInitMaxSpots) run the standalone
    initializer in front of the fit -- per host chunk, or into a stream-ordered scratch buffer for
    device batches -- with the same results as explicit standalone inits; mixed tame / general spots."""
    import torch

    P = sf.batch_engine.ENGINES[engine]
    count = 40_001
    im = _sim(sf, W, H, count, seed=5 + W * H, model=4 if P == 4 else 3).astype(np.float32)
    im[::7] += np.float32(0.25)  # general (non-integer) spots interleaved with tame ones
    grid = sf.PixelGrid(W, H)
    ref = sf.fit_batch(im, _standalone_inits(sf, im, W, H, P), grid=grid, engine=engine)
    _same(sf.fit_batch(im, grid=grid, engine=engine), ref, f"host f32 {W}x{H} {engine}")
    _same(sf.fit_batch(torch.from_numpy(im).cuda(), grid=grid, engine=engine), ref, f"device f32 {W}x{H} {engine}")
    ti = np.round(im[1::7])  # integer spots only for the u16 paths
    u = ti.astype(np.uint16)
    ref16 = sf.fit_batch(ti, _standalone_inits(sf, ti, W, H, P), grid=grid, engine=engine)
    _same(sf.fit_batch(u, grid=grid, engine=engine), ref16, f"host u16 {W}x{H} {engine}")
    big = np.concatenate([u] * 4)
    refb = sf.fit_batch(big.astype(np.float32), _standalone_inits(sf, big.astype(np.float32), W, H, P), grid=grid,
                        engine=engine)
    _same(sf.fit_batch(torch.from_numpy(big).cuda(), grid=grid, engine=engine), refb, f"device u16 {W}x{H} {engine}")


@pytest.mark.parametrize("W,H,engine", [(15, 15, "implicit3"), (32, 32, "implicit3"), (5, 40, "implicit3"),
                                        (21, 21, "elliptical"), (13, 11, "explicit5")])
def test_fused_init_integer_and_general_paths(sf, W, H, engine):
    """The fused initializer's exact integer path (every pixel an integer in [0, 2^20]) and its
    general f64 path, interleaved spot by spot inside one batch (so groups of one warp take
    different paths): fractional pixels, integers above 2^20, -0.0, tiny and negative values."""
    P = sf.batch_engine.ENGINES[engine]
    count = 4000
    im = _sim(sf, W, H, count, seed=77 + W, model=4 if P == 4 else 3).astype(np.float32)
    rng = np.random.default_rng(W * H)
    k = np.arange(count) % 8
    im[k == 1] += np.float32(0.5)  # fractional
    im[k == 2] *= np.float32(4096.0)  # integers above 2^20 (the peak)
    im[k == 3, 0] = np.float32(-0.0)
    im[k == 4, rng.integers(0, W * H)] = np.float32(1e-30)
    im[k == 5] -= np.float32(3.0)  # negative background
    im[k == 6] = np.float32(1048576.0)  # exactly 2^20: still the integer path
    grid = sf.PixelGrid(W, H)
    ref = sf.fit_batch(im, _standalone_inits(sf, im, W, H, P), grid=grid, engine=engine)
    _same(sf.fit_batch(im, grid=grid, engine=engine), ref, f"mixed paths {W}x{H} {engine}")
    oi, oa = oinit.estimate_initial_batch_np(im, W, H, 0.3, float(max(W, H)), 3 if P == 5 else P)
    si, sa = sf.estimate_initial_batch(im, 3 if P == 5 else P, grid=grid)
    assert bits_equal(si, oi) and bits_equal(sa, oa)


def test_fused_init_matches_oracle_end_to_end(sf, oracle_lib):
    """inits=None against the C oracle driven by the oracle initializer (oracle/initializer.py)."""
    W = H = 15
    count = 3000
    im = _sim(sf, W, H, count, seed=4321)
    im[0] = 3.0  # constant image: centre (0, 0), sigma_min
    oi, _ = oinit.estimate_initial_batch(im, W, H, 0.3, 15.0, 3)
    ref = oracle_lib.fit_batch(im, oi, W, H, lm.LMConfig.for_grid(W, H))
    _same(sf.fit_batch(im, grid=sf.PixelGrid(W, H)), ref, "fused vs oracle")


def test_fused_init_multichunk_pageable_and_shards(sf):
    """A batch of several host chunks, pageable and pinned, and two shards (devices=[0, 0]):
    no inits cross PCIe, results unchanged."""
    import torch

    W = H = 15
    count = 70_000
    im = _sim(sf, W, H, count, seed=55)
    ref = sf.fit_batch(im, _standalone_inits(sf, im, W, H, 3), grid=sf.PixelGrid(W, H))
    a = sf.fit_batch(im, grid=sf.PixelGrid(W, H))
    assert a.stats["n_chunks"] >= 4
    _same(a, ref, "pageable")
    _same(sf.fit_batch(torch.from_numpy(im).pin_memory().numpy(), grid=sf.PixelGrid(W, H)), ref, "pinned")
    _same(sf.fit_batch(im, grid=sf.PixelGrid(W, H), devices=[0, 0]), ref, "two shards")


def _nonfinite_images(sf, W, H, count, seed):
    im = _sim(sf, W, H, count, seed=seed).copy()
    rng = np.random.default_rng(seed)
    kinds = np.arange(count) % 9
    pix = rng.integers(0, W * H, count)
    for kind, val in ((1, np.nan), (2, np.inf), (3, -np.inf)):
        rows = np.nonzero(kinds == kind)[0]
        im[rows, pix[rows]] = np.float32(val)
    im[kinds == 4, 0] = np.float32(np.nan)  # smoothed_0 NaN: the scan never leaves index 0
    im[kinds == 5] = np.float32(np.nan)  # all NaN
    rows = np.nonzero(kinds == 6)[0]  # +inf and -inf in one window: inf - inf = NaN in the sum
    im[rows, pix[rows]] = np.float32(np.inf)
    im[rows, (pix[rows] + 1) % (W * H)] = np.float32(-np.inf)
    im[kinds == 7] = np.float32(-np.inf)
    im[kinds == 8, : W * H // 2] = np.float32(-1e30)
    return im


@pytest.mark.parametrize("W,H", [(15, 15), (32, 32), (5, 3), (1, 7)])
def test_initializer_nonfinite_matches_oracle(sf, W, H):
    """The standalone initializer follows numpy's NaN semantics exactly (first maximum
    by a strict ">" scan from smoothed_0, min propagating NaN)."""
    im = _nonfinite_images(sf, W, H, 900, seed=W * 31 + H)
    for model in (3, 4):
        ini, amps = sf.estimate_initial_batch(im, model, grid=sf.PixelGrid(W, H))
        oi, oa = oinit.estimate_initial_batch(im, W, H, 0.3, float(max(W, H)), model)
        assert bits_equal(ini, oi), (W, H, model, np.nonzero(~np.all(ini.view(np.uint32) == oi.view(np.uint32), 1)))
        assert bits_equal(amps, oa), (W, H, model)


@pytest.mark.parametrize("W,H,engine", [(15, 15, "implicit3"), (32, 32, "implicit3"), (21, 21, "elliptical"),
                                        (13, 11, "explicit5")])
def test_fused_init_nonfinite_matches_standalone(sf, W, H, engine):
    """Non-finite pixels with inits=None: InvalidInput results carrying the fused estimate,
    bitwise the standalone initializer's (so the batch API returns the same rows either way)."""
    P = sf.batch_engine.ENGINES[engine]
    im = _nonfinite_images(sf, W, H, 1800, seed=3 * W + H)
    grid = sf.PixelGrid(W, H)
    ref = sf.fit_batch(im, _standalone_inits(sf, im, W, H, P), grid=grid, engine=engine)
    _same(sf.fit_batch(im, grid=grid, engine=engine), ref, f"nonfinite {W}x{H} {engine}")


def test_standalone_initializer_u16_input(sf):
    """estimate_initial_batch on uint16 counts: widened before the launch."""
    import torch

    W = H = 15
    im = _sim(sf, W, H, 500, seed=6)
    u = im.astype(np.uint16)
    a = sf.estimate_initial_batch(im, 3, grid=sf.PixelGrid(W, H))
    for src in (u, torch.from_numpy(u), torch.from_numpy(u).cuda()):
        b = sf.estimate_initial_batch(src, 3, grid=sf.PixelGrid(W, H))
        assert bits_equal(a[0], b[0]) and bits_equal(a[1], b[1])
    with pytest.raises(TypeError):
        sf.batch_engine.estimate_initial_device(torch.from_numpy(u).cuda(), sf.PixelGrid(W, H), 3)


def test_mixed_host_device_arguments_fail(sf):
    """sf_fit_batch checks every pointer: device images with a host output
    array, or host images with a device output array, return an error instead of
    writing through the wrong address space."""
    import torch

    W = H = 9
    count = 64
    L = sf._lib.lib()
    ccfg = sf.FitConfig().to_c(sf.PixelGrid(W, H), 3)
    d_im = torch.zeros((count, W * H), device="cuda") + 5.0
    h_im = np.full((count, W * H), 5.0, np.float32)
    h = dict(par=np.empty((count, 3), np.float32), f=np.empty((3, count), np.float32), u8=np.empty((2, count), np.uint8))
    d = dict(par=torch.empty((count, 3), device="cuda"), f=torch.empty((3, count), device="cuda"),
             u8=torch.empty((2, count), dtype=torch.uint8, device="cuda"))
    st = sf._lib.sf_stats()
    dev = (ctypes.c_int32 * 1)(0)
    rc = L.sf_fit_batch(d_im.data_ptr(), W, H, count, None, ctypes.byref(ccfg), d["par"].data_ptr(),
                        d["f"][0].data_ptr(), d["f"][1].data_ptr(), d["f"][2].data_ptr(), h["u8"][0].ctypes.data,
                        d["u8"][1].data_ptr(), dev, 1, ctypes.byref(st))
    assert rc != 0 and b"mixed" in L.sf_last_error()
    rc = L.sf_fit_batch(h_im.ctypes.data, W, H, count, None, ctypes.byref(ccfg), h["par"].ctypes.data,
                        d["f"][0].data_ptr(), h["f"][1].ctypes.data, h["f"][2].ctypes.data, h["u8"][0].ctypes.data,
                        h["u8"][1].ctypes.data, dev, 1, ctypes.byref(st))
    assert rc != 0 and b"mixed" in L.sf_last_error()
    # all-device and all-host calls still work, and agree
    rc = L.sf_fit_batch(d_im.data_ptr(), W, H, count, None, ctypes.byref(ccfg), d["par"].data_ptr(),
                        d["f"][0].data_ptr(), d["f"][1].data_ptr(), d["f"][2].data_ptr(), d["u8"][0].data_ptr(),
                        d["u8"][1].data_ptr(), dev, 1, ctypes.byref(st))
    assert rc == 0, L.sf_last_error()
    rc = L.sf_fit_batch(h_im.ctypes.data, W, H, count, None, ctypes.byref(ccfg), h["par"].ctypes.data,
                        h["f"][0].ctypes.data, h["f"][1].ctypes.data, h["f"][2].ctypes.data, h["u8"][0].ctypes.data,
                        h["u8"][1].ctypes.data, dev, 1, ctypes.byref(st))
    assert rc == 0, L.sf_last_error()
    assert bits_equal(h["par"], d["par"].cpu().numpy()) and bits_equal(h["u8"], d["u8"].cpu().numpy())


def test_device_entry_restores_current_device(sf):
    """The device entry points launch on the device owning the pixels and leave the
    caller's current device unchanged; the host pipeline restores it too."""
    import torch

    W = H = 11
    im = _sim(sf, W, H, 300, seed=3)
    cur = torch.cuda.current_device()
    sf.fit_batch(torch.from_numpy(im).cuda(), grid=sf.PixelGrid(W, H))
    sf.fit_batch(im, grid=sf.PixelGrid(W, H), devices=[0])
    assert torch.cuda.current_device() == cur


def test_work_slots_never_shared_under_load(sf, oracle_lib):
    """300 launches in flight at once on 8 streams (more than the 256 stream slots of the
    work-claim pool): the pool waits for a finished slot instead of sharing a counter, so
    every spot of every launch is fitted exactly once."""
    import torch

    W = H = 15
    count = 600
    im = _sim(sf, W, H, count, seed=31)
    ini = oinit.estimate_initial_batch(im, W, H, 0.3, 15.0, 3)[0]
    ref = oracle_lib.fit_batch(im, ini, W, H, lm.LMConfig.for_grid(W, H))
    L = sf._lib.lib()
    ccfg = sf.FitConfig().to_c(sf.PixelGrid(W, H), 3)
    d_im = torch.from_numpy(im).cuda()
    d_ini = torch.from_numpy(ini).cuda()
    streams = [torch.cuda.Stream() for _ in range(8)]
    launches = 300
    outs = []
    for k in range(launches):
        b = dict(par=torch.full((count, 3), -1.0, device="cuda"), fl=torch.empty((3, count), device="cuda"),
                 u8=torch.full((2, count), 255, dtype=torch.uint8, device="cuda"))
        st = streams[k % len(streams)]
        sf._lib.check(L.sf_fit_batch_device(d_im.data_ptr(), W, H, count, d_ini.data_ptr(), ctypes.byref(ccfg),
                                            b["par"].data_ptr(), b["fl"][0].data_ptr(), b["fl"][1].data_ptr(),
                                            b["fl"][2].data_ptr(), b["u8"][0].data_ptr(), b["u8"][1].data_ptr(), None,
                                            st.cuda_stream))
        outs.append(b)
    torch.cuda.synchronize()
    for b in outs[:: 37] + outs[-3:]:
        assert bits_equal(b["par"].cpu().numpy(), ref["params"])
        assert bits_equal(b["u8"][0].cpu().numpy(), ref["status"])
        assert bits_equal(b["u8"][1].cpu().numpy(), ref["iterations"])


def test_tame_division_exhaustive(sf):
    """The initializer's integer-path division (sf_init_core.cuh:tame_div: multiply by the
    rounded reciprocal, one exact-residual correction) equals IEEE s / c for every integer
    s in [0, 9 * 2^20] and every truncated-window count c in {1, 2, 3, 4, 6, 9}."""
    import torch

    m = torch.zeros(1, dtype=torch.int64, device="cuda")
    sf._lib.check(sf._lib.lib().sf_debug_tame_div_device(m.data_ptr(), torch.cuda.current_stream().cuda_stream))
    assert int(m.item()) == 0


def test_standalone_initializer_geometry_sweep(sf):
    """The standalone initializer (sf_init.cu) on every grid width 1..32 against the vectorised
    oracle: one column per lane, row-segmented columns (W < L / 2), two adjacent columns per lane
    (L < W <= 2L) and the general wide path; tame (integer) and general (fractional) spots mixed;
    odd counts (the last staging window pokes out of the array) and a device batch that starts
    4 bytes past a 16-byte boundary (every window takes the element-copy path at its edges)."""
    import torch

    rng = np.random.default_rng(11)
    for W in range(1, 33):
        for H in (1, 2, 3, 7, 16, 31, 32):
            count = 301
            im = _sim(sf, W, H, count, seed=1000 + 33 * W + H).astype(np.float32)
            im[rng.random(count) < 0.3] += np.float32(0.5)  # general-path spots
            grid = sf.PixelGrid(W, H)
            oi, oa = oinit.estimate_initial_batch_np(im, W, H, 0.3, float(max(W, H)), 3)
            si, sa = sf.estimate_initial_batch(im, 3, grid=grid)
            assert bits_equal(si, oi) and bits_equal(sa, oa), (W, H, "host")
            flat = torch.zeros(count * W * H + 1, dtype=torch.float32, device="cuda")
            flat[1:] = torch.from_numpy(im.reshape(-1)).cuda()
            di, da = sf.estimate_initial_batch(flat[1:].view(count, H, W), 3, grid=grid)
            assert bits_equal(np.asarray(di), oi) and bits_equal(np.asarray(da), oa), (W, H, "offset device")


def test_standalone_initializer_u16_geometry_sweep(sf):
    """The 16-bit instantiation of the standalone initializer (integer column walk, 8-per-chunk M
    count) on every grid width: device uint16 batches above the fused-initializer size without
    inits run it in front of the fit; the results equal the float32 batch's (whose initializer the
    f32 sweep pins to the oracle) bit for bit."""
    import torch

    count = 16_400  # > sf_launch.h:kFusedInitMaxSpots
    for W in range(1, 33):
        for H in (3, 16, 32):
            grid = sf.PixelGrid(W, H)
            d, _ = sf.simulate_batch_device(sf.SimConfig(width=W, height=H, count=count, seed=7 * W + H))
            d = d.reshape(count, W * H)
            a = sf.fit_batch(d, grid=grid)
            b = sf.fit_batch(torch.from_numpy(d.cpu().numpy().astype(np.uint16)).cuda(), grid=grid)
            _same(b, a, f"u16 device {W}x{H}")
