"""Check the native float32 rendering (csrc/sf_csv.cpp, sf_format_f32) against numpy's Dragon4
(np.format_float_positional(unique=True, trim='-'), io_formats.fmt32) over a range of float32 bit
patterns: every positive finite value when run with --all (the sign only prepends '-').

    python tools/csv_format_check.py --all --procs 8      # exhaustive: 2^31 - 2^23 patterns
    python tools/csv_format_check.py --start 0x3f800000 --count 1000000
"""
from __future__ import annotations

import argparse
import ctypes
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BLOCK = 1 << 18


def native(bits: np.ndarray) -> list:
    from paper_2106_02045_b200 import _lib

    v = np.ascontiguousarray(bits.view(np.float32))
    cap = 80 * len(v) + 80
    buf = ctypes.create_string_buffer(cap)
    n = ctypes.c_int64(0)
    _lib.check(_lib.lib().sf_format_f32(v.ctypes.data, len(v), buf, cap, ctypes.byref(n)))
    return buf.raw[: n.value].decode().split("\n")[:-1]


def check_block(lo: int, hi: int):
    bits = np.arange(lo, hi, dtype=np.uint64).astype(np.uint32)
    got = native(bits)
    fmt = np.format_float_positional
    bad = []
    for b, g in zip(bits.view(np.float32), got):
        w = fmt(b, unique=True, trim="-")
        if w != g:
            bad.append((int(b.view(np.uint32)), g, w))
            if len(bad) > 20:
                break
    return hi - lo, bad


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--all", action="store_true")
    ap.add_argument("--start", type=lambda s: int(s, 0), default=0)
    ap.add_argument("--count", type=int, default=1 << 20)
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    a = ap.parse_args(argv)
    lo, hi = (1, 0x7F800000) if a.all else (a.start, a.start + a.count)
    jobs = [(s, min(hi, s + BLOCK)) for s in range(lo, hi, BLOCK)]
    t0 = time.time()
    done, bad = 0, []
    with mp.Pool(a.procs) as pool:
        for k, (n, b) in enumerate(pool.imap_unordered(_star, jobs, chunksize=4)):
            done += n
            bad += b
            if k % 512 == 0:
                print(f"{done:,} checked, {len(bad)} mismatches, {time.time() - t0:.0f} s", flush=True)
    print(f"range [{lo:#x}, {hi:#x}): {done:,} float32 patterns, {len(bad)} mismatches, "
          f"{time.time() - t0:.0f} s on {a.procs} processes")
    for b in bad[:20]:
        print(f"  {b[0]:#010x}: native {b[1]!r} numpy {b[2]!r}")
    return 1 if bad else 0


def _star(j):
    return check_block(*j)


if __name__ == "__main__":
    sys.exit(main())
