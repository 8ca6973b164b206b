"""SPEC.md acceptance criteria 1-4 (Table 1 and Fig. 8) on the GPU at the SPEC's sample size
(>= 50,000 spots per setting): simulate -> initialise -> fit -> assess, all on the device.  The 1e6-spot
run of every criterion, including the stop-reason mix of criterion 5, is tools/acceptance.py
(profiles/r02_acceptance.json)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sf():
    import paper_2106_02045_b200 as sf

    sf._lib.require_gpu()
    return sf


@pytest.fixture(scope="module")
def runs(sf):
    import acceptance as acc

    return {
        "400:40": acc.run_setting(sf, 9, 400.0, 40.0, 50_000, 4040),
        "1600:40": acc.run_setting(sf, 9, 1600.0, 40.0, 50_000, 16040, engines=("implicit3", "explicit5")),
        "1600:0": acc.run_setting(sf, 9, 1600.0, 0.0, 50_000, 16000),
    }


def test_table1_400_40(runs):
    import acceptance as acc

    a = runs["400:40"]["implicit3"]["accuracy"]
    want = acc.TABLE1["400:40"]
    for got, w in ((a["position_median"], want[0]), (a["position_mean"], want[1]), (a["position_std"], want[2]),
                   (a["sigma_median"], want[3])):
        assert acc.within(got, w), (got, w)


def test_table1_1600_40(runs):
    import acceptance as acc

    a = runs["1600:40"]["implicit3"]["accuracy"]
    want = acc.TABLE1["1600:40"]
    for got, w in ((a["position_median"], want[0]), (a["position_mean"], want[1]), (a["sigma_median"], want[3])):
        assert acc.within(got, w), (got, w)


def test_shot_noise_ratio_1600_0(runs):
    r = runs["1600:0"]["implicit3"]["accuracy"]["position_mean"] * 1600 ** 0.5
    assert 1.0 <= r <= 1.2, r


def test_implicit_needs_fewer_iterations_than_explicit5(runs):
    i3, e5 = runs["1600:40"]["implicit3"]["iterations"], runs["1600:40"]["explicit5"]["iterations"]
    assert i3["mode"] in (4, 5) and i3["mean"] < e5["mean"], (i3, e5)
    f = runs["1600:40"]["implicit3"]["frac"]
    assert f["min_delta_family"] > 0.5 and f["max_iterations"] <= 0.001 and f["not_converged"] == 0.0
