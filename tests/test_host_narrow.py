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


@pytest.mark.parametrize("offset", [0, 2, 30])
def test_narrowing_into_an_unaligned_destination(offset):
    """Aligned destinations take streaming stores, others plain ones: same values either way."""
    rng = np.random.default_rng(offset)
    a = rng.integers(0, 65536, (1 << 20) + 9).astype(np.float32)
    buf = np.empty(a.size + 64, np.uint16)
    out = buf[offset // 2:offset // 2 + a.size]
    rc = _lib.lib().sf_debug_narrow_u16(a.ctypes.data, a.size, out.ctypes.data, 3)
    assert rc == 1 and np.array_equal(out.astype(np.float32), a)


@pytest.mark.parametrize("pos", [0, 4095, 4096, 1 << 20, (1 << 20) + 4097, 3 * (1 << 20)])
def test_early_exit_refuses_across_thread_pieces(pos):
    """A non-integer value anywhere in a multi-threaded pass (other pieces stop early) refuses it."""
    a = np.arange(3 * (1 << 20) + 11, dtype=np.float32) % 60000
    a[pos] = 0.5
    ok, _ = narrow(a, threads=4)
    assert not ok


@pytest.mark.parametrize("nbytes", [0, 1, 31, 4095, 4096, 4097, (4 << 20) * 3 + 129])
@pytest.mark.parametrize("dst_off", [0, 8, 32])
@pytest.mark.parametrize("src_off", [0, 3])
def test_staging_copy(nbytes, dst_off, src_off):
    """The pageable staging copy (sf::par_copy: threads, streaming stores when the destination is
    32-byte aligned) copies every byte."""
    rng = np.random.default_rng(nbytes)
    src = rng.integers(0, 256, nbytes + 64, dtype=np.uint8)
    dst = np.zeros(nbytes + 128, np.uint8)
    base = dst.ctypes.data
    d0 = (-base) % 64 + dst_off
    rc = _lib.lib().sf_debug_par_copy(base + d0, src.ctypes.data + src_off, nbytes, 4)
    assert rc == 0
    assert np.array_equal(dst[d0:d0 + nbytes], src[src_off:src_off + nbytes])
    assert not dst[:d0].any() and not dst[d0 + nbytes:].any()
