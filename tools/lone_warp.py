"""One fit launch with one warp per SM sub-partition (148 CTAs x 4 warps, 1184 15x15 spots):
the latency view of the fit kernel for ncu source-level stall sampling.

    ncu --set full --import-source on -k regex:fit_kernel -c 1 -o gpurun_out/lone python tools/lone_warp.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_02045_b200 as sf  # noqa: E402
from paper_2106_02045_b200 import _lib  # noqa: E402

W = H = 15
n = 148 * 8
im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=n, seed=3))
ini, _ = sf.estimate_initial_batch(im, 3)
grid = sf.PixelGrid(W, H)
cfg = sf.FitConfig().to_c(grid, 3)
d_im = torch.from_numpy(im.reshape(n, -1)).cuda()
d_ini = torch.from_numpy(ini).cuda()
par = torch.empty((n, 3), device="cuda")
fl = torch.empty((3, n), device="cuda")
u8 = torch.empty((2, n), dtype=torch.uint8, device="cuda")
L = _lib.lib()
for _ in range(2):
    _lib.check(L.sf_fit_batch_device(d_im.data_ptr(), W, H, n, d_ini.data_ptr(), ctypes.byref(cfg), par.data_ptr(),
                                     fl[0].data_ptr(), fl[1].data_ptr(), fl[2].data_ptr(), u8[0].data_ptr(),
                                     u8[1].data_ptr(), None, None))
torch.cuda.synchronize()
print("lone-warp fit done")
