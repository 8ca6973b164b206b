"""The spotfit.model function surface (reference pkg/src/spotfit/model.py:168-315):
profile, profile_and_gradient, profile_gradient, alpha_beta, model_values,
residuals, chi_squared, gradient_sums, coefficient_gradients, chi_gradient --
each called by its reference name and compared bit for bit with the outputs of
the reference itself (tests/golden/model_pixels_golden.npz, made by
tests/golden/make_golden.py from the imported reference), including on
profile / gradient arrays that did not come from the profile and on a
SingularProfile case.  The CPU test pins the oracle restatement to the same
fixtures; the GPU tests run the product (csrc/sf_model.cu via sf_model_*)."""
import numpy as np
import pytest

from conftest import bits_equal, load_golden
from oracle import model_np

GOLD = load_golden("model_pixels_golden.npz")
CASES = range(len(GOLD["kind"]))


def _case(m, i):
    W, H = (int(v) for v in GOLD["shape"][i])
    N = W * H
    grid = m.PixelGrid(W, H)
    img = m.SpotImage(grid, GOLD["image"][i][:N])
    return W, H, N, grid, img, GOLD["f"][i][:N], GOLD["fgrad"][i][:N]


def _check_chain(m, i):
    W, H, N, grid, img, f, fg = _case(m, i)
    p = m.ShapeParams(*GOLD["params"][i])
    assert bits_equal(m.profile(p, grid), GOLD["f_profile"][i][:N])
    if GOLD["kind"][i] == 0:
        f2, fg2 = m.profile_and_gradient(p, grid)
        assert bits_equal(f2, f) and bits_equal(fg2, fg)
        assert bits_equal(m.profile_gradient(p, grid), fg)
    if GOLD["singular"][i]:
        with pytest.raises(m.SingularProfile):
            m.alpha_beta(f, img)
        return
    amps, sums = m.alpha_beta(f, img)
    assert amps.alpha == GOLD["alpha"][i] and amps.beta == GOLD["beta"][i]
    assert bits_equal(np.array([sums.f_sum, sums.g_sum, sums.ff_sum, sums.fg_sum, sums.denom]), GOLD["sums"][i])
    assert sums.n == N
    assert bits_equal(np.asarray(m.model_values(f, amps), np.float32), GOLD["h"][i][:N])
    assert bits_equal(np.asarray(m.residuals(img, f, amps), np.float32), GOLD["r"][i][:N])
    assert np.float32(m.chi_squared(img, f, amps)) == GOLD["chi"][i]
    gs = m.gradient_sums(f, fg, img, sums)
    assert bits_equal(np.stack([gs.df, gs.dff, gs.dfg, gs.gamma]), GOLD["gsums"][i])
    da, db = m.coefficient_gradients(sums, gs, amps)
    assert bits_equal(np.asarray(da), GOLD["dalpha"][i]) and bits_equal(np.asarray(db), GOLD["dbeta"][i])
    grad, d = m.chi_gradient(img, f, fg, amps, (da, db))
    assert bits_equal(np.asarray(grad), GOLD["grad"][i]) and bits_equal(np.asarray(d, np.float32), GOLD["dmat"][i][:N])


@pytest.mark.parametrize("i", CASES)
def test_oracle_model_functions_match_reference(i):
    _check_chain(model_np, i)


@pytest.mark.gpu
@pytest.mark.parametrize("i", CASES)
def test_gpu_model_functions_match_reference(i):
    import paper_2106_02045_b200 as sf

    _check_chain(sf, i)


@pytest.mark.gpu
def test_gpu_model_batch_functions_match_reference():
    """The batched forms (one kernel per function over all spots of one grid) give the
    single-spot results; rows are independent."""
    import paper_2106_02045_b200 as sf

    shapes = sorted({tuple(int(v) for v in s) for s in GOLD["shape"]})
    for W, H in shapes:
        idx = [i for i in CASES if tuple(int(v) for v in GOLD["shape"][i]) == (W, H)]
        N = W * H
        grid = sf.PixelGrid(W, H)
        g = GOLD["image"][idx][:, :N]
        f = GOLD["f"][idx][:, :N]
        fg = GOLD["fgrad"][idx][:, :N]
        fp = sf.profile_batch(GOLD["params"][idx], grid).cpu().numpy()
        assert bits_equal(fp, GOLD["f_profile"][idx][:, :N])
        a, b, sums, sing = (t.cpu().numpy() for t in sf.alpha_beta_batch(f, g))
        ok = sing == 0
        assert bits_equal(sing, GOLD["singular"][idx].astype(np.int32))
        assert bits_equal(a[ok], GOLD["alpha"][idx][ok]) and bits_equal(sums[ok], GOLD["sums"][idx][ok])
        assert np.all(np.isnan(a[~ok]))
        chi, h, r = (t.cpu().numpy() for t in sf.chi_squared_batch(g, f, a, b, values=True))
        assert bits_equal(chi[ok], GOLD["chi"][idx][ok]) and bits_equal(h[ok], GOLD["h"][idx][ok][:, :N])
        assert bits_equal(r[ok], GOLD["r"][idx][ok][:, :N])
        gs = sf.gradient_sums_batch(f, fg, g, sums).cpu().numpy()
        assert bits_equal(gs[ok], GOLD["gsums"][idx][ok])
        da, db, sing2 = (t.cpu().numpy() for t in sf.coefficient_gradients_batch(sums, gs, a, b, N))
        assert bits_equal(sing2, sing)
        assert bits_equal(da[ok], GOLD["dalpha"][idx][ok]) and bits_equal(db[ok], GOLD["dbeta"][idx][ok])
        grad, d = (t.cpu().numpy() for t in sf.chi_gradient_batch(g, f, fg, a, b, da, db))
        assert bits_equal(grad[ok], GOLD["grad"][idx][ok]) and bits_equal(d[ok], GOLD["dmat"][idx][ok][:, :N])


@pytest.mark.gpu
def test_gpu_elliptical_model_functions_match_oracle():
    """P = 4 (x, y, sigma_x, sigma_y, no reference): every function against the
    oracle's elliptical restatement (pinned by tests/test_elliptical_pin.py)."""
    import paper_2106_02045_b200 as sf

    for W, H in ((21, 21), (15, 15), (7, 5), (32, 32)):
        im, tr = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=3, seed=W * 3 + H, model=4))
        for s in range(3):
            g = im[s].reshape(-1)
            pe = sf.EllipticalParams(*tr[s][:4])
            po = model_np.EllipticalParams(*tr[s][:4])
            grid, ogrid = sf.PixelGrid(W, H), model_np.PixelGrid(W, H)
            img, oimg = sf.SpotImage(grid, g), model_np.SpotImage(ogrid, g)
            f, fg = sf.profile_and_gradient(pe, grid)
            of, ofg = model_np.profile_and_gradient(po, ogrid)
            assert bits_equal(f, of) and bits_equal(fg, ofg)
            amps, sums = sf.alpha_beta(f, img)
            oamps, osums = model_np.alpha_beta(of, oimg)
            assert amps.alpha == oamps.alpha and sums.denom == osums.denom
            gs = sf.gradient_sums(f, fg, img, sums)
            ogs = model_np.gradient_sums(of, ofg, oimg, osums)
            assert bits_equal(gs.gamma, ogs.gamma) and bits_equal(gs.dfg, ogs.dfg)
            cg = sf.coefficient_gradients(sums, gs, amps)
            ocg = model_np.coefficient_gradients(osums, ogs, oamps)
            assert bits_equal(cg[0], ocg[0]) and bits_equal(cg[1], ocg[1])
            grad, d = sf.chi_gradient(img, f, fg, amps, cg)
            ograd, od = model_np.chi_gradient(oimg, of, ofg, oamps, ocg)
            assert bits_equal(grad, ograd) and bits_equal(d, od)


@pytest.mark.gpu
def test_gpu_model_functions_argument_errors():
    import paper_2106_02045_b200 as sf

    grid = sf.PixelGrid(5, 5)
    img = sf.SpotImage(grid, np.ones(25, np.float32))
    with pytest.raises(ValueError):
        sf.alpha_beta(np.ones(24, np.float32), img)
    with pytest.raises(sf.SingularProfile):
        sf.alpha_beta(np.full(25, 0.5, np.float32), img)
    with pytest.raises(ValueError):
        sf.profile_batch(np.ones((2, 5), np.float32), grid)
