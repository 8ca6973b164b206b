"""Per-call latency of the public fit_batch from host memory for small batches (the overhead
regime of the paper's Fig. 2 / SPEC bench module): Python front end vs the C-ABI call alone vs
the device-resident entry point, median of many calls.

    python tools/call_overhead.py [count ...]
"""
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def med(fn, n=300):
    for _ in range(10):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)) * 1e6


def main():
    import torch

    import paper_2106_02045_b200 as sf
    from paper_2106_02045_b200 import _lib

    counts = [int(c) for c in sys.argv[1:]] or [1, 10, 100, 1000]
    L = _lib.lib()
    out = []
    for n in counts:
        W = H = 15
        im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=n, seed=9))
        flat = np.ascontiguousarray(im.reshape(n, W * H))
        ini, _ = sf.estimate_initial_batch(flat, 3, grid=sf.PixelGrid(W, H))
        grid = sf.PixelGrid(W, H)
        cfg = sf.FitConfig().to_c(grid, 3)
        par = np.empty((n, 3), np.float32)
        f = np.empty((3, n), np.float32)
        u8 = np.empty((2, n), np.uint8)
        dev = (ctypes.c_int32 * 1)(0)
        p = lambda a: a.ctypes.data  # noqa: E731

        def capi():
            _lib.check(L.sf_fit_batch(p(flat), W, H, n, p(ini), ctypes.byref(cfg), p(par), f[0].ctypes.data,
                                      f[1].ctypes.data, f[2].ctypes.data, u8[0].ctypes.data, u8[1].ctypes.data, dev, 1,
                                      None))

        d_im = torch.from_numpy(flat).cuda()
        d_ini = torch.from_numpy(ini).cuda()
        d_par = torch.empty((n, 3), device="cuda")
        d_f = torch.empty((3, n), device="cuda")
        d_u8 = torch.empty((2, n), dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream().cuda_stream

        def device():
            _lib.check(L.sf_fit_batch_device(d_im.data_ptr(), W, H, n, d_ini.data_ptr(), ctypes.byref(cfg),
                                              d_par.data_ptr(), d_f[0].data_ptr(), d_f[1].data_ptr(), d_f[2].data_ptr(),
                                              d_u8[0].data_ptr(), d_u8[1].data_ptr(), None, st))
            torch.cuda.current_stream().synchronize()

        out.append({"spots": n, "fit_batch_us": med(lambda: sf.fit_batch(flat, ini, grid=grid)),
                    "fit_batch_no_inits_us": med(lambda: sf.fit_batch(flat, grid=grid)),
                    "c_abi_us": med(capi), "device_entry_us": med(device)})
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
