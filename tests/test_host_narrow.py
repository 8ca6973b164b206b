"""The host pipeline's lossless f32 -> u16 narrowing (csrc/sf_host_narrow.cpp, sf_debug_narrow_u16):
a chunk crosses PCIe as u16 only when every pixel is an integer in [0, 65535] with a clear sign bit,
and then the u16 values are exactly the pixels (the fit kernel widens them back exactly)."""

import numpy as np
import pytest

from paper_2106_02045_b200 import _lib


def narrow(a, threads=4):
    a = np.ascontiguousarray(a, np.float32)
    out = np.empty(a.size, np.uint16)
    rc = _lib.lib().sf_debug_narrow_u16(a.ctypes.data, a.size, out.ctypes.data, threads)
    assert rc in (0, 1)
    return rc == 1, out


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 33, 4096 * 257 + 5, 3 * (1 << 20) + 7])
def test_integer_chunks_narrow_exactly(n):
    rng = np.random.default_rng(n)
    a = rng.integers(0, 65536, n).astype(np.float32)
    ok, out = narrow(a)
    assert ok and np.array_equal(out.astype(np.float32), a)


@pytest.mark.parametrize("bad", [-0.0, -1.0, 0.5, 65536.0, 65535.5, 1e-45, 1.17549435e-38, np.inf, -np.inf, np.nan,
                                 1e30, 4294967296.0])
@pytest.mark.parametrize("pos", [0, 7, 15, 16, 1000, -1])
def test_any_other_value_refuses_the_chunk(bad, pos):
    a = np.arange(2000, dtype=np.float32) % 65536
    a[pos] = bad
    ok, _ = narrow(a, threads=3)
    assert not ok


def test_edges_of_the_range():
    a = np.float32([0.0, 1.0, 65535.0, 65534.0, 255.0, 256.0, 32768.0] * 5)
    ok, out = narrow(a)
    assert ok and np.array_equal(out.astype(np.float32), a)
