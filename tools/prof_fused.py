"""Minimal driver for ncu: one standalone initializer launch and one fused-init fit launch
(15x15, HBM-resident).  python tools/prof_fused.py [count]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2106_02045_b200 as sf

    count = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
    W = H = 15
    grid = sf.PixelGrid(W, H)
    L = sf._lib.lib()
    d_img, _ = sf.simulate_batch_device(sf.SimConfig(width=W, height=H, count=count, seed=5))
    d_img = d_img.reshape(count, -1).contiguous()
    d_ini = sf.batch_engine.estimate_initial_device(d_img, grid, 3)
    par = torch.empty((count, 3), device="cuda")
    fl = torch.empty((3, count), device="cuda")
    u8 = torch.empty((2, count), dtype=torch.uint8, device="cuda")
    ccfg = sf.FitConfig().to_c(grid, 3)
    st = torch.cuda.current_stream().cuda_stream
    for ini in (None, d_ini):
        sf._lib.check(L.sf_fit_batch_device(d_img.data_ptr(), W, H, count, None if ini is None else ini.data_ptr(),
                                            ctypes.byref(ccfg), par.data_ptr(), fl[0].data_ptr(), fl[1].data_ptr(),
                                            fl[2].data_ptr(), u8[0].data_ptr(), u8[1].data_ptr(), None, st))
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
