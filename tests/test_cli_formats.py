"""SPB1 / ParamsCSV formats, assess, and the CLI.
CPU tests; the GPU `fit` end-to-end test is marked gpu."""
import json
import os

import numpy as np
import pytest

from conftest import bits_equal, load_golden


def test_spb1_roundtrip_and_layout(tmp_path):
    from paper_2106_02045_b200.io_formats import read_spb1, write_spb1

    rng = np.random.default_rng(0)
    a = rng.standard_normal((17, 5, 7)).astype(np.float32)
    p = tmp_path / "x.spb"
    write_spb1(str(p), a)
    # SPEC.md:520 field layout (4+2+2+2+4 = 14-byte header; SPEC.md:521's "12 +" is inconsistent with it)
    assert os.path.getsize(p) == 14 + 4 * 17 * 5 * 7
    raw = open(p, "rb").read()
    assert raw[:4] == b"SPB1" and raw[4:6] == b"\x01\x00" and raw[6:8] == b"\x07\x00" and raw[8:10] == b"\x05\x00"
    assert raw[10:14] == (17).to_bytes(4, "little")
    b, W, H = read_spb1(str(p))
    assert (W, H) == (7, 5) and bits_equal(np.asarray(b), a)
    write_spb1(str(p), np.zeros((0, 3, 3), np.float32))  # count = 0 is valid
    z, _, _ = read_spb1(str(p))
    assert z.shape == (0, 3, 3)


@pytest.mark.parametrize("mutate,offset", [(lambda b: b"SPB2" + b[4:], 0), (lambda b: b[:4] + b"\x02\x00" + b[6:], 4),
                                           (lambda b: b[:-4], None), (lambda b: b[:8], 8)])
def test_spb1_malformed_reports_offset(tmp_path, mutate, offset):
    from paper_2106_02045_b200.io_formats import MalformedSPB1, read_spb1, write_spb1

    p = tmp_path / "x.spb"
    write_spb1(str(p), np.ones((3, 4, 4), np.float32))
    data = mutate(open(p, "rb").read())
    open(p, "wb").write(data)
    with pytest.raises(MalformedSPB1) as e:
        read_spb1(str(p))
    if offset is not None:
        assert e.value.offset == offset


def test_params_csv_roundtrip(tmp_path):
    from paper_2106_02045_b200.batch_engine import BatchResult
    from paper_2106_02045_b200.io_formats import read_params_csv, write_params_csv

    fit = load_golden("fit_golden.npz")
    r = BatchResult(fit["15x15_params"], fit["15x15_alpha"], fit["15x15_beta"], fit["15x15_nchi2"],
                    fit["15x15_status"], fit["15x15_iterations"])
    p = tmp_path / "f.csv"
    write_params_csv(str(p), r)
    head = open(p).readline().strip()
    assert head == "index,x,y,sigma,alpha,beta,status,iterations,nchi2"
    back = read_params_csv(str(p))
    assert bits_equal(back["params"], r.params) and bits_equal(back["alpha"], r.alpha)
    assert bits_equal(back["beta"], r.beta) and bits_equal(back["nchi2"], r.nchi2)
    assert np.array_equal(back["stop"], r.status & 7) and np.array_equal(back["iterations"], r.iterations)
    assert np.array_equal(back["index"], np.arange(len(r.alpha)))


def test_shortest_float_format():
    from paper_2106_02045_b200.io_formats import fmt32

    assert fmt32([0.1, 1.0, 2.5e-8, 3.4028235e38]) == ["0.1", "1", "0.000000025", "340282350000000000000000000000000000000"]
    v = np.float32(np.random.default_rng(3).standard_normal(1000))
    assert all(np.float32(s) == x for s, x in zip(fmt32(v), v))


def test_assess_statistics():
    from paper_2106_02045_b200.assess import accuracy, expected_error_ratio, iteration_stats

    truth = np.array([[1.0, 2.0, 1.5, 10.0, 1.0], [3.0, 3.0, 1.0, 10.0, 1.0]], np.float32)
    s = accuracy(truth[:, :3], np.array([1, 2], np.uint8), truth)
    assert s.position_median == s.position_mean == s.position_std == 0.0
    p = truth[:, :3].copy()
    p[0, 0] += 0.15
    p[1, 2] = -1.1  # sigma error uses |sigma^|
    s = accuracy(p, np.array([1, 3], np.uint8), truth)  # second fit NotConverged -> excluded
    assert s.n_excluded == 1 and s.n_fits == 1
    assert abs(s.position_mean - 0.05) < 1e-6
    assert abs(expected_error_ratio(s, 400.0) - 0.05 * 20) < 1e-6
    h = iteration_stats(np.array([1, 1 | 0x80, 2, 3], np.uint8), np.array([5, 5, 4, 20]))
    assert h["mode"] == 5 and h["stop_reasons"]["MinDelta"] == 2 and h["no_improvement"] == 1
    assert sum(h["histogram"]) == 4


def test_cli_simulate_deterministic_and_limits(tmp_path):
    from paper_2106_02045_b200.cli import main

    a, b = tmp_path / "a.spb", tmp_path / "b.spb"
    ta, tb = tmp_path / "a.csv", tmp_path / "b.csv"
    assert main(["simulate", "--size", "9", "--count", "50", "--seed", "42", "--out", str(a), "--truth", str(ta)]) == 0
    assert main(["simulate", "--size", "9", "--count", "50", "--seed", "42", "--out", str(b), "--truth", str(tb)]) == 0
    assert open(a, "rb").read() == open(b, "rb").read() and open(ta).read() == open(tb).read()
    assert main(["simulate", "--size", "33", "--count", "1", "--out", str(a)]) == 2
    assert main(["simulate", "--size", "9", "--count", "0", "--out", str(a)]) == 0
    assert os.path.getsize(a) == 14
    assert main(["fit", "--bogus"]) == 2


def test_cli_fit_malformed_and_engine(tmp_path):
    from paper_2106_02045_b200.cli import main

    p = tmp_path / "bad.spb"
    open(p, "wb").write(b"NOPE" + b"\x00" * 20)
    assert main(["fit", "--in", str(p), "--out", str(tmp_path / "o.csv")]) == 4
    assert main(["fit", "--in", str(tmp_path / "missing.spb"), "--out", str(tmp_path / "o.csv")]) == 3
    assert main(["fit", "--in", str(p), "--out", str(tmp_path / "o.csv"), "--engine", "bogus"]) == 2


@pytest.mark.gpu
def test_cli_simulate_fit_assess_end_to_end(tmp_path, oracle_lib):
    """simulate | fit | assess: CSV rows bit-equal the oracle and
    >= 99% of fits stop MinDelta/MinStep."""
    from oracle import initializer as oinit
    from oracle import lm
    from paper_2106_02045_b200.cli import main
    from paper_2106_02045_b200.io_formats import read_params_csv, read_spb1

    spb, truth, fits, rep = (tmp_path / n for n in ("s.spb", "t.csv", "f.csv", "r.json"))
    assert main(["simulate", "--size", "9", "--count", "1000", "--seed", "42", "--out", str(spb),
                 "--truth", str(truth)]) == 0
    assert main(["fit", "--in", str(spb), "--out", str(fits)]) == 0
    got = read_params_csv(str(fits))
    im, W, H = read_spb1(str(spb))
    im = np.asarray(im).reshape(1000, -1)
    ini, _ = oinit.estimate_initial_batch(im, W, H, 0.3, 9.0)
    ref = oracle_lib.fit_batch(im, ini, W, H, lm.LMConfig.for_grid(W, H))
    assert bits_equal(got["params"], ref["params"]) and bits_equal(got["alpha"], ref["alpha"])
    assert np.array_equal(got["stop"], ref["status"] & 7)
    assert np.mean(np.isin(got["stop"], [1, 2])) >= 0.99
    assert main(["assess", "--fits", str(fits), "--truth", str(truth), "--report", str(rep), "--signal", "400"]) == 0
    r = json.load(open(rep))
    assert r["accuracy"]["n_fits"] + r["accuracy"]["n_excluded"] == 1000
    assert 0.02 < r["accuracy"]["position_median"] < 0.1  # Table 1 scale


@pytest.mark.gpu
def test_cli_flags_column_feeds_assess(tmp_path):
    """fit --flags writes status & 0xf8; assess then counts the no-improvement stops (acceptance
    criterion 5), which the SPEC header alone cannot carry."""
    from paper_2106_02045_b200.cli import main
    from paper_2106_02045_b200.io_formats import read_params_csv

    spb, truth, fits, fits2, rep, rep2 = (tmp_path / n for n in ("s.spb", "t.csv", "f.csv", "g.csv", "r.json",
                                                               "q.json"))
    assert main(["simulate", "--size", "9", "--count", "3000", "--seed", "5", "--signal", "1600", "--out",
                 str(spb), "--truth", str(truth)]) == 0
    assert main(["fit", "--in", str(spb), "--out", str(fits), "--flags"]) == 0
    assert main(["fit", "--in", str(spb), "--out", str(fits2)]) == 0
    got = read_params_csv(str(fits))
    assert "flags" in got and int(((got["flags"] & 0x80) != 0).sum()) > 0
    assert main(["assess", "--fits", str(fits), "--truth", str(truth), "--report", str(rep)]) == 0
    assert main(["assess", "--fits", str(fits2), "--truth", str(truth), "--report", str(rep2)]) == 0
    r, r2 = json.load(open(rep)), json.load(open(rep2))
    assert r["iterations"]["no_improvement"] == int(((got["flags"] & 0x80) != 0).sum())
    assert r2["iterations"]["no_improvement"] is None  # unavailable without the column, not a false 0
    assert r["accuracy"] == r2["accuracy"]


def test_bench_default_plan_is_the_papers():
    """S = 4..32 x batches 10/100/1000/10000 -> 29 * 4 = 116 entries, repeated
    200x, 20x, 10x and once."""
    from paper_2106_02045_b200.cli import CliError, bench_plan, build_parser

    a = build_parser().parse_args(["bench"])
    plan = bench_plan(a.sizes, a.batches, a.repeats)
    assert len(plan) == 116
    assert {(b, r) for _, b, r in plan} == {(10, 200), (100, 20), (1000, 10), (10000, 1)}
    assert sorted({s for s, _, _ in plan}) == list(range(4, 33))
    with pytest.raises(CliError):
        bench_plan("33", "10")


@pytest.mark.gpu
def test_cli_bench_report(tmp_path):
    """run_bench report identities: fits/s * time = batch, pixels/s = fits/s * S^2."""
    from paper_2106_02045_b200.cli import main

    rep, csv = tmp_path / "b.json", tmp_path / "b.csv"
    assert main(["bench", "--sizes", "9,16", "--batches", "10,1000", "--repeats", "3,2", "--report", str(rep),
                 "--csv", str(csv)]) == 0
    r = json.load(open(rep))
    assert len(r["entries"]) == 4 and "B200" in r["machine"]
    for e in r["entries"]:
        assert abs(e["fits_per_s"] * e["seconds_per_call"] - e["batch"]) < 1e-6 * e["batch"]
        assert abs(e["pixels_per_s"] - e["fits_per_s"] * e["size"] ** 2) < 1e-6 * e["pixels_per_s"]
    assert len(open(csv).read().splitlines()) == 5
