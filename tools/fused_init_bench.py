"""Kernel-only cost of the fused initializer: sf_fit_batch_device with explicit inits vs
inits=NULL (f32 and u16 pixels), and the standalone initializer (sf_estimate_initial_device)
in GB/s of pixels read.  HBM-resident inputs, CUDA events, median of repeats.

    python tools/fused_init_bench.py [--count 1000000]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2106_02045_b200 as sf

    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    L = sf._lib.lib()
    out = {}
    for (W, H, P) in ((15, 15, 3), (11, 11, 3), (21, 21, 4), (32, 32, 3)):
        count = a.count if W * H <= 441 else a.count // 2
        grid = sf.PixelGrid(W, H)
        d_img, _ = sf.simulate_batch_device(sf.SimConfig(width=W, height=H, count=count, seed=5, model=P))
        d_img = d_img.reshape(count, -1).contiguous()
        d_u16 = d_img.to(torch.int32).to(torch.uint16)
        d_ini = sf.batch_engine.estimate_initial_device(d_img, grid, P)
        par = torch.empty((count, P), device="cuda")
        fl = torch.empty((3, count), device="cuda")
        u8 = torch.empty((2, count), dtype=torch.uint8, device="cuda")
        ccfg = sf.FitConfig().to_c(grid, P)
        st = torch.cuda.current_stream().cuda_stream
        b = sf.FitConfig().resolved_bounds(grid)

        def fit(img, ini, u16=False):
            fn = L.sf_fit_batch_device_u16 if u16 else L.sf_fit_batch_device
            sf._lib.check(fn(img.data_ptr(), W, H, count, None if ini is None else ini.data_ptr(), ctypes.byref(ccfg),
                             par.data_ptr(), fl[0].data_ptr(), fl[1].data_ptr(), fl[2].data_ptr(), u8[0].data_ptr(),
                             u8[1].data_ptr(), None, st))

        def init():
            sf._lib.check(L.sf_estimate_initial_device(d_img.data_ptr(), W, H, count, P, b.sigma_min, b.sigma_max,
                                                       d_ini.data_ptr(), None, st))

        def t(fn):
            fn()
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            return float(np.median(ts))

        r = {"count": count, "explicit_f32_ms": t(lambda: fit(d_img, d_ini)),
             "fused_f32_ms": t(lambda: fit(d_img, None)),
             "explicit_u16_ms": t(lambda: fit(d_u16, d_ini, True)), "fused_u16_ms": t(lambda: fit(d_u16, None, True)),
             "standalone_init_ms": t(init)}
        r["fused_overhead_f32"] = r["fused_f32_ms"] / r["explicit_f32_ms"] - 1
        r["fused_overhead_u16"] = r["fused_u16_ms"] / r["explicit_u16_ms"] - 1
        r["standalone_init_GBps"] = count * W * H * 4 / (r["standalone_init_ms"] * 1e-3) / 1e9
        out[f"{W}x{H}_P{P}"] = r
        print(json.dumps({f"{W}x{H}_P{P}": r}), flush=True)


if __name__ == "__main__":
    main()
