"""Native ParamsCSV / truth-CSV I/O (csrc/sf_csv.cpp) against the numpy statement of the rendering
(io_formats.fmt32 = np.format_float_positional(unique=True, trim='-')) and the
round-trip property.  The exhaustive check over every positive finite float32 is
tools/csv_format_check.py --all (profiles/r02_csv_format_exhaustive.txt)."""
import ctypes

import numpy as np
import pytest

from paper_2106_02045_b200 import _lib
from paper_2106_02045_b200.io_formats import (fmt32, read_params_csv, read_truth_csv, write_params_csv,
                                              write_truth_csv)


def native_fmt(values) -> list:
    v = np.ascontiguousarray(values, np.float32)
    cap = 80 * len(v) + 80
    buf = ctypes.create_string_buffer(cap)
    n = ctypes.c_int64(0)
    _lib.check(_lib.lib().sf_format_f32(v.ctypes.data, len(v), buf, cap, ctypes.byref(n)))
    return buf.raw[: n.value].decode().split("\n")[:-1]


def edge_values() -> np.ndarray:
    bits = [0, 1, 2, 3, 0x007FFFFF, 0x00800000, 0x00800001, 0x7F7FFFFF, 0x7F800000, 0x7FC00000, 0x3F800000,
            0x3DCCCCCD, 0x4B800000, 0x4B7FFFFF]
    for e in range(0, 255):  # every binade: first, second, middle and last mantissa
        for m in (0, 1, 0x400000, 0x7FFFFE, 0x7FFFFF):
            bits.append((e << 23) | m)
    bits = np.array(bits, np.uint32)
    bits = np.concatenate([bits, bits | np.uint32(0x80000000)])
    dec = np.float32([1e-45, 1e-38, 1e-10, 1e-7, 0.1, 0.2, 0.3, 1.0, 2.5, 100.0, 123456.7, 1e7, 16777216.0,
                      16777217.0, 3.4028235e38, 9.999999e-1, 5e-324, 1.17549435e-38, 2.0 ** -126, 2.0 ** -149,
                      0.000025, 1e21, 1e22, 1e23, 8.589973e9, 2.4414062e-4])
    return np.concatenate([bits.view(np.float32), dec, -dec])


def test_native_rendering_equals_numpy_on_edges():
    v = edge_values()
    got, want = native_fmt(v), fmt32(v)
    bad = [(hex(int(np.float32(x).view(np.uint32))), g, w) for x, g, w in zip(v, got, want) if g != w]
    assert not bad, bad[:10]


def test_native_rendering_equals_numpy_on_random_bits():
    bits = np.random.default_rng(2106).integers(0, 2 ** 32, 200_000, dtype=np.uint64).astype(np.uint32)
    v = bits.view(np.float32)
    got, want = native_fmt(v), fmt32(v)
    bad = [(hex(int(b)), g, w) for b, g, w in zip(bits, got, want) if g != w]
    assert not bad, bad[:10]


def test_native_rendering_round_trips_fit_like_values():
    rng = np.random.default_rng(5)
    v = np.float32(np.concatenate([rng.uniform(0, 15, 50_000), rng.lognormal(0, 3, 50_000),
                                   rng.standard_normal(50_000) * 1e-3]))
    got = native_fmt(v)
    assert np.array_equal(np.array(got, dtype=np.float32).view(np.uint32), v.view(np.uint32))


class _Res:
    def __init__(self, n, P, rng):
        self.params = np.float32(rng.uniform(-3, 20, (n, P)))
        self.params[::97] = np.nan
        self.alpha = np.float32(rng.lognormal(5, 2, n))
        self.beta = np.float32(rng.standard_normal(n) * 40)
        self.nchi2 = np.float32(rng.lognormal(0, 1, n))
        self.nchi2[3::101] = np.inf
        self.status = rng.integers(0, 5, n).astype(np.uint8) | (rng.integers(0, 2, n).astype(np.uint8) << 7)
        self.status[::53] |= 0x40
        self.iterations = rng.integers(0, 21, n).astype(np.uint8)


@pytest.mark.parametrize("P,flags", [(3, False), (3, True), (4, True), (5, False)])
def test_params_csv_round_trip_bitwise(tmp_path, P, flags):
    n = 20_011
    r = _Res(n, P, np.random.default_rng(P + 10 * flags))
    p = tmp_path / "fits.csv"
    write_params_csv(str(p), r, first_index=7, flags=flags, threads=3)
    head = open(p).readline().strip().split(",")
    assert head[:4] == ["index", "x", "y", "sigma"] and ("flags" in head) == flags
    back = read_params_csv(str(p), threads=5)
    K = 4 if P == 4 else 3
    assert np.array_equal(back["params"].view(np.uint32), r.params[:, :K].view(np.uint32))
    for k in ("alpha", "beta", "nchi2"):
        assert np.array_equal(back[k].view(np.uint32), getattr(r, k).view(np.uint32)), k
    assert np.array_equal(back["stop"], r.status & 7) and np.array_equal(back["iterations"], r.iterations)
    assert np.array_equal(back["index"], np.arange(7, 7 + n))
    if flags:
        assert np.array_equal(back["flags"], r.status & 0xF8)
    # the rows are exactly the numpy rendering
    lines = open(p).read().splitlines()[1:]
    i = 1234
    want = [str(7 + i)] + [fmt32([r.params[i, k]])[0] for k in range(K)] + [
        fmt32([r.alpha[i]])[0], fmt32([r.beta[i]])[0],
        ["MaxError", "MinDelta", "MinStep", "NotConverged", "MaxIterations"][r.status[i] & 7],
        str(r.iterations[i]), fmt32([r.nchi2[i]])[0]] + ([str(r.status[i] & 0xF8)] if flags else [])
    assert lines[i] == ",".join(want)


def test_truth_csv_round_trip_and_empty(tmp_path):
    t = np.float32(np.random.default_rng(1).uniform(0, 50, (999, 6)))
    p = tmp_path / "t.csv"
    write_truth_csv(str(p), t)
    assert open(p).readline().strip() == "index,x,y,sigma,sigma_y,alpha,beta"
    assert np.array_equal(read_truth_csv(str(p)).view(np.uint32), t.view(np.uint32))
    e = _Res(0, 3, np.random.default_rng(0))
    write_params_csv(str(p), e)
    assert open(p).read() == "index,x,y,sigma,alpha,beta,status,iterations,nchi2\n"
    back = read_params_csv(str(p))
    assert back["params"].shape == (0, 3) and back["alpha"].shape == (0,)


def test_malformed_rows_raise(tmp_path):
    p = tmp_path / "bad.csv"
    for body in ("0,1,2,3,4,5,MinDelta,4,1.5\n1,1,2,x,4,5,MinDelta,4,1.5\n",
                 "0,1,2,3,4,5,Bogus,4,1.5\n", "0,1,2,3,4,5,MinDelta,4\n", "0,1,2,3,4,5,MinDelta,4,1.5,9\n",
                 "0,1,2,3,4,5,MinDelta,400,1.5\n"):
        p.write_text("index,x,y,sigma,alpha,beta,status,iterations,nchi2\n" + body)
        with pytest.raises(ValueError, match="malformed row"):
            read_params_csv(str(p))
    p.write_text("index,x,y,alpha\n0,1,2,3\n")
    with pytest.raises(ValueError, match="missing columns"):
        read_params_csv(str(p))


def test_crlf_and_blank_lines_are_accepted(tmp_path):
    p = tmp_path / "crlf.csv"
    p.write_bytes(b"index,x,y,sigma,alpha,beta,status,iterations,nchi2\r\n"
                  b"0,1.5,2,3,4,5,MinStep,4,1.25\r\n\r\n1,0.1,2,3,4,5,MaxIterations,20,nan\r\n")
    back = read_params_csv(str(p))
    assert back["params"][1, 0] == np.float32(0.1) and list(back["stop"]) == [2, 4] and np.isnan(back["nchi2"][1])
