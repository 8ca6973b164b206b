"""Pins the oracle (numpy restatement oracle/model_np.py, LM oracle/lm.py, C
twin oracle/spotfit_oracle.c) bit-for-bit against fixtures produced by the
REFERENCE model.py (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import bits_equal, load_golden
from oracle import lm, model_np

MODEL = load_golden("model_golden.npz")
FIT = load_golden("fit_golden.npz")
FIT_KEYS = sorted({k.rsplit("_", 1)[0] for k in FIT.files if k.endswith("_images")})


def _cases():
    for i, (W, H) in enumerate(MODEL["shape"]):
        yield i, int(W), int(H)


def test_model_np_matches_reference_golden():
    for i, W, H in _cases():
        N = W * H
        grid = model_np.PixelGrid(W, H)
        img = model_np.SpotImage(grid, MODEL["image"][i][:N])
        p = model_np.ShapeParams(*MODEL["params"][i])
        f, fg = model_np.profile_and_gradient(p, grid)
        if MODEL["has_pixels"][i]:
            assert bits_equal(f, MODEL["f"][i][:N].astype(np.float32))
            assert bits_equal(fg, MODEL["fgrad"][i][:N].astype(np.float32))
            assert bits_equal(model_np.profile(p, grid), MODEL["f_profile"][i][:N].astype(np.float32))
        if MODEL["singular"][i]:
            with pytest.raises(model_np.SingularProfile):
                model_np.alpha_beta(f, img)
            continue
        amps, sums = model_np.alpha_beta(f, img)
        assert amps.alpha == MODEL["alpha"][i] and amps.beta == MODEL["beta"][i]
        for k, v in (("F", sums.f_sum), ("G", sums.g_sum), ("FF", sums.ff_sum), ("FG", sums.fg_sum),
                     ("denom", sums.denom)):
            assert v == MODEL[k][i], (i, k)
        assert model_np.chi_squared(img, f, amps) == MODEL["chi"][i]
        gs = model_np.gradient_sums(f, fg, img, sums)
        cg = model_np.coefficient_gradients(sums, gs, amps)
        grad, d = model_np.chi_gradient(img, f, fg, amps, cg)
        for k, v in (("dF", gs.df), ("dFF", gs.dff), ("dFG", gs.dfg), ("gamma", gs.gamma), ("dalpha", cg[0]),
                     ("dbeta", cg[1]), ("grad", grad)):
            assert bits_equal(np.asarray(v), MODEL[k][i]), (i, k)
        jtj = [float((d[:, j] * d[:, k]).sum(dtype=np.float64)) for j in range(3) for k in range(j, 3)]
        assert bits_equal(np.array(jtj), MODEL["jtj"][i])


def test_c_oracle_eval_matches_reference_golden(oracle_lib):
    for i, W, H in _cases():
        N = W * H
        r = oracle_lib.eval_batch(MODEL["image"][i][:N][None, :], MODEL["params"][i][None, :], W, H, threads=1)[0]
        assert bool(r["singular"]) == bool(MODEL["singular"][i]), i
        if r["singular"]:
            continue
        assert r["alpha"] == MODEL["alpha"][i] and r["beta"] == MODEL["beta"][i] and r["chi"] == MODEL["chi"][i]
        for k in ("F", "G", "FF", "FG", "denom"):
            assert r[k] == MODEL[k][i], (i, k)
        for k in ("dF", "dFF", "dFG", "gamma", "dalpha", "dbeta"):
            assert bits_equal(r[k][:3], MODEL[k][i]), (i, k)
        assert bits_equal(r["rhs"][:3] * -2.0, MODEL["grad"][i])
        assert bits_equal(r["jtj"][:6], MODEL["jtj"][i])


def _fit_case(key):
    W, H = (int(v) for v in key.split("x"))
    return W, H, FIT[f"{key}_images"], FIT[f"{key}_inits"]


def _check_fit(res, key, n=None):
    sl = slice(0, n)
    for k in ("params", "alpha", "beta", "nchi2", "status", "iterations"):
        assert bits_equal(np.asarray(res[k])[sl], FIT[f"{key}_{k}"][sl]), (key, k)


@pytest.mark.parametrize("key", FIT_KEYS)
def test_c_oracle_fit_matches_reference_golden(oracle_lib, key):
    W, H, im, ini = _fit_case(key)
    res = oracle_lib.fit_batch(im, ini, W, H, lm.LMConfig.for_grid(W, H), threads=4)
    _check_fit(res, key)


@pytest.mark.parametrize("key", ["15x15", "7x5", "21x21"])
def test_numpy_lm_over_restatement_matches_reference_golden(key):
    W, H, im, ini = _fit_case(key)
    n = 60
    res = lm.fit_batch_arrays(model_np, im[:n], ini[:n], W, H, lm.LMConfig.for_grid(W, H))
    _check_fit(res, key, n)
    assert np.array_equal(res["n_g"], FIT[f"{key}_n_g"][:n]) and np.array_equal(res["n_t"], FIT[f"{key}_n_t"][:n])


def test_solve_step_golden(oracle_lib):
    for J, r, lam, d, ok in zip(FIT["solve_jtj"], FIT["solve_rhs"], FIT["solve_lam"], FIT["solve_delta"],
                                FIT["solve_ok"]):
        got = lm.solve_step(J, r, lam)
        assert (got is not None) == bool(ok)
        cok, cd = oracle_lib.solve(J, r, lam)
        assert cok == bool(ok)
        if ok:
            assert bits_equal(np.array(got), d) and bits_equal(cd, d)
