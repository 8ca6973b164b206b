"""ParamsCSV throughput: rows/s of the native writer and reader
(csrc/sf_csv.cpp) on fit-like results, against the numpy-statement writer (fmt32 per value) on a
small sample.  Writes to a temporary directory (tmpfs when /dev/shm exists).

    python tools/csv_bench.py [--rows 10000000] [--threads 0]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class Res:
    def __init__(self, n, rng):
        self.params = np.float32(np.stack([rng.uniform(0, 15, n), rng.uniform(0, 15, n), rng.uniform(1, 2, n)], 1))
        self.alpha = np.float32(rng.normal(400, 20, n))
        self.beta = np.float32(rng.normal(40, 2, n))
        self.nchi2 = np.float32(rng.lognormal(0, 0.1, n))
        self.status = rng.integers(1, 3, n).astype(np.uint8)
        self.iterations = rng.integers(3, 8, n).astype(np.uint8)


def main(argv=None):
    from paper_2106_02045_b200.io_formats import fmt32, read_params_csv, write_params_csv

    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args(argv)
    r = Res(a.rows, np.random.default_rng(0))
    base = "/dev/shm" if os.path.isdir("/dev/shm") else None
    with tempfile.TemporaryDirectory(dir=base) as d:
        p = os.path.join(d, "fits.csv")
        write_params_csv(p, r, threads=a.threads)  # warm the page cache / allocator
        t0 = time.perf_counter()
        write_params_csv(p, r, threads=a.threads)
        tw = time.perf_counter() - t0
        size = os.path.getsize(p)
        t0 = time.perf_counter()
        back = read_params_csv(p, threads=a.threads)
        tr = time.perf_counter() - t0
        ok = bool(np.array_equal(back["params"].view(np.uint32), r.params.view(np.uint32)) and
                  np.array_equal(back["nchi2"].view(np.uint32), r.nchi2.view(np.uint32)))
    n_py = 20000
    t0 = time.perf_counter()
    for k in range(3):
        fmt32(r.params[:n_py, k])
    for arr in (r.alpha, r.beta, r.nchi2):
        fmt32(arr[:n_py])
    tpy = time.perf_counter() - t0
    out = {"rows": a.rows, "bytes": size, "dir": base or tempfile.gettempdir(), "threads": a.threads or os.cpu_count(),
           "write_rows_per_s": a.rows / tw, "write_s": tw, "read_rows_per_s": a.rows / tr, "read_s": tr,
           "round_trip_bitwise": ok, "numpy_fmt32_rows_per_s": n_py / tpy}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
