"""Pins the elliptical (x0, y0, sigma_x, sigma_y) model, which has no reference
counterpart (SPEC.md:152 lists it as a non-goal), by the
two independent checks SURVEY 8(c) names:

  * central finite differences of an f64 evaluation of the same model
    (exact Gaussian, closed-form alpha/beta of Eq. 6) against the oracle's
    analytic f32 partials, amplitude gradients (Eq. 8), chi^2 gradient (Eq. 9)
    and the Gauss-Newton normal matrix J^T J;
  * the identity profile_ellip(x, y, s, s) == profile(x, y, s), bitwise for f,
    the x/y partials, F, FF, FG, alpha, beta and chi^2, with
    d/dsigma_x + d/dsigma_y == d/dsigma up to f32 rounding.

The oracle (oracle/model_np.py) is the checker for the GPU's P = 4 kernels, so
these tests are what make a sign or factor error shared by oracle and kernel
visible.  CPU tests, plus one GPU test of the identity on the kernel itself.
"""
import numpy as np
import pytest

from conftest import bits_equal
from oracle import lm, model_np

STEP = 1e-4


def _f64_model(g, W, H, p):
    """f64 evaluation: f_i, alpha, beta, h_i = alpha f_i + beta, chi^2 (Eq. 6, no rounding to f32)."""
    x = np.arange(W * H) % W
    y = np.arange(W * H) // W
    x0, y0, sx, sy = (float(v) for v in p)
    f = np.exp(-0.5 * (((x - x0) / sx) ** 2 + ((y - y0) / sy) ** 2))
    n = f.size
    F, G, FF, FG = f.sum(), g.sum(), (f * f).sum(), (f * g).sum()
    D = n * FF - F * F
    a = (n * FG - F * G) / D
    b = (G * FF - F * FG) / D
    h = a * f + b
    return f, a, b, h, float(((g - h) ** 2).sum())


def _fd(fun, p, k):
    hi = np.array(p, np.float64)
    lo = np.array(p, np.float64)
    hi[k] += STEP
    lo[k] -= STEP
    return (np.asarray(fun(hi)) - np.asarray(fun(lo))) / (2 * STEP)


def _cases():
    import paper_2106_02045_b200 as sf  # the host generator only (no GPU needed)

    out = []
    for W, H in ((21, 21), (15, 15), (13, 9), (32, 32)):
        im, tr = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=6, seed=W * 101 + H, model=4))
        rng = np.random.default_rng(W + H)
        for s in range(6):
            x, y, sx, sy = (float(v) for v in tr[s][:4])
            p = model_np.EllipticalParams(x + rng.normal(0, 0.4), y + rng.normal(0, 0.4), sx * rng.uniform(0.8, 1.25),
                                          sy * rng.uniform(0.8, 1.25))
            out.append((W, H, im[s].reshape(-1).astype(np.float32), p))
    return out


CASES = _cases()


@pytest.mark.parametrize("case", range(len(CASES)))
def test_elliptical_derivatives_match_finite_differences(case):
    W, H, g, p = CASES[case]
    grid = model_np.PixelGrid(W, H)
    img = model_np.SpotImage(grid, g)
    pa = p.as_array().astype(np.float64)
    f, fg = model_np.profile_and_gradient(p, grid)
    amps, sums = model_np.alpha_beta(f, img)
    gs = model_np.gradient_sums(f, fg, img, sums)
    da, db = model_np.coefficient_gradients(sums, gs, amps)
    grad, d = model_np.chi_gradient(img, f, fg, amps, (da, db))
    g64 = g.astype(np.float64)
    jtj = np.array([[float((d[:, j] * d[:, k]).sum(dtype=np.float64)) for k in range(4)] for j in range(4)])  # f32 products
    dfd = np.empty((W * H, 4))
    for k in range(4):
        fd_f = _fd(lambda q: _f64_model(g64, W, H, q)[0], pa, k)
        scale = np.abs(fd_f).max()
        assert np.abs(fg[:, k] - fd_f).max() <= 1e-3 * scale + 1e-6, ("df/dp", k)
        fd_a = float(_fd(lambda q: _f64_model(g64, W, H, q)[1], pa, k))
        fd_b = float(_fd(lambda q: _f64_model(g64, W, H, q)[2], pa, k))
        assert abs(da[k] - fd_a) <= 1e-3 * abs(fd_a) + 1e-3 * abs(amps.alpha) * 1e-2, ("dalpha", k, da[k], fd_a)
        assert abs(db[k] - fd_b) <= 1e-3 * abs(fd_b) + 1e-3 * max(abs(amps.beta), 1.0) * 1e-2, ("dbeta", k)
        fd_chi = float(_fd(lambda q: _f64_model(g64, W, H, q)[4], pa, k))
        chi = _f64_model(g64, W, H, pa)[4]
        assert abs(grad[k] - fd_chi) <= 1e-3 * abs(fd_chi) + 1e-4 * chi, ("dchi2/dp", k, grad[k], fd_chi)
        dfd[:, k] = _fd(lambda q: _f64_model(g64, W, H, q)[3], pa, k)  # model derivative d_ik = dh_i/dp_k
        assert np.abs(d[:, k] - dfd[:, k]).max() <= 1e-3 * np.abs(dfd[:, k]).max(), ("d_ik", k)
    jtj_fd = dfd.T @ dfd
    assert np.all(np.abs(jtj - jtj_fd) <= 2e-3 * np.sqrt(np.outer(np.diag(jtj_fd), np.diag(jtj_fd)))), "J^T J"
    # the LM oracle's packed normal system is the same J^T J and rhs = -grad/2
    e = lm.g_eval(model_np, img, list(p.as_array()))
    packed = [jtj[j, k] for j in range(4) for k in range(j, 4)]
    assert bits_equal(np.asarray(e.jtj), np.asarray(packed)) and bits_equal(np.asarray(e.rhs), -0.5 * grad)


@pytest.mark.parametrize("case", range(len(CASES)))
def test_elliptical_reduces_to_symmetric_when_sigmas_equal(case):
    W, H, g, p = CASES[case]
    grid = model_np.PixelGrid(W, H)
    img = model_np.SpotImage(grid, g)
    s = p.sigma_x
    pe = model_np.EllipticalParams(p.x, p.y, s, s)
    ps = model_np.ShapeParams(p.x, p.y, s)
    fe, ge = model_np.profile_and_gradient(pe, grid)
    fs, gsym = model_np.profile_and_gradient(ps, grid)
    assert bits_equal(fe, fs) and bits_equal(model_np.profile(pe, grid), model_np.profile(ps, grid))
    assert bits_equal(ge[:, 0], gsym[:, 0]) and bits_equal(ge[:, 1], gsym[:, 1])
    # d/dsigma_x + d/dsigma_y = d/dsigma (u^2 f/s + v^2 f/s = q f/s), up to f32 rounding
    tot = ge[:, 2].astype(np.float64) + ge[:, 3]
    assert np.abs(tot - gsym[:, 2]).max() <= 4e-7 * max(1.0, np.abs(gsym[:, 2]).max())
    ae, se = model_np.alpha_beta(fe, img)
    as_, ss = model_np.alpha_beta(fs, img)
    assert ae == as_ and se == ss
    assert model_np.chi_squared(img, fe, ae) == model_np.chi_squared(img, fs, as_)
    # x / y amplitude gradients and rhs entries are the same sums of the same f32 terms
    ee = lm.g_eval(model_np, img, list(pe.as_array()))
    es = lm.g_eval(model_np, img, list(ps.as_array()))
    assert ee.rhs[0] == es.rhs[0] and ee.rhs[1] == es.rhs[1]
    assert ee.jtj[0] == es.jtj[0] and ee.jtj[1] == es.jtj[1] and ee.jtj[4] == es.jtj[3]  # xx, xy, yy
    assert abs(ee.rhs[2] + ee.rhs[3] - es.rhs[2]) <= 1e-5 * (abs(es.rhs[2]) + abs(ee.rhs[2]) + abs(ee.rhs[3]))


def test_c_oracle_elliptical_equals_numpy_oracle():
    """The C twin (the GPU's large-sample checker) reproduces model_np's elliptical evaluation bitwise."""
    from oracle import oracle_c

    for W, H, g, p in CASES[::3]:
        rec = oracle_c.eval_batch(g[None, :], p.as_array()[None, :], W, H)[0]
        e = lm.g_eval(model_np, model_np.SpotImage(model_np.PixelGrid(W, H), g), list(p.as_array()))
        assert rec["chi"] == np.float32(e.chi) and rec["alpha"] == np.float32(e.alpha)
        assert bits_equal(np.asarray(rec["rhs"][:4]), np.asarray(e.rhs))
        assert bits_equal(np.asarray(rec["jtj"][:10]), np.asarray(e.jtj))


@pytest.mark.gpu
def test_gpu_elliptical_reduces_to_symmetric():
    """The P = 4 kernel at (x, y, s, s) against the P = 3 kernel at (x, y, s): identical profile
    sums, amplitudes, chi^2, x/y gradient entries; sigma entries add up."""
    import paper_2106_02045_b200 as sf

    for W, H in ((21, 21), (15, 15), (32, 32), (7, 5)):
        im, tr = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=500, seed=W * H, model=3))
        p3 = np.ascontiguousarray(tr[:, :3])
        p4 = np.ascontiguousarray(np.concatenate([tr[:, :3], tr[:, 2:3]], axis=1))
        r3 = sf.evaluate_batch(im.reshape(500, -1), p3, W, H)
        r4 = sf.evaluate_batch(im.reshape(500, -1), p4, W, H)
        for k in ("alpha", "beta", "chi", "F", "G", "FF", "FG", "denom", "singular"):
            assert bits_equal(r3[k], r4[k]), (W, H, k)
        for k in ("dF", "dFF", "dFG", "gamma", "dalpha", "dbeta", "rhs"):
            assert bits_equal(r3[k][:, :2], r4[k][:, :2]), (W, H, k)
        assert bits_equal(r3["jtj"][:, [0, 1, 3]], r4["jtj"][:, [0, 1, 4]]), (W, H)
        tot = r4["rhs"][:, 2] + r4["rhs"][:, 3]
        assert np.all(np.abs(tot - r3["rhs"][:, 2]) <= 1e-5 * (np.abs(r3["rhs"][:, 2]) + np.abs(r4["rhs"][:, 2])
                                                               + np.abs(r4["rhs"][:, 3]) + 1e-30))
