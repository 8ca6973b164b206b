"""GPU initializer throughput (sf_estimate_initial_device on HBM-resident 15x15 spots)."""
import sys
import os
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_02045_b200 as sf  # noqa: E402

W = H = int(sys.argv[1]) if len(sys.argv) > 1 else 15
n = 1_000_000
im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=n, seed=3))
d = torch.from_numpy(im).cuda()
for _ in range(3):
    sf.estimate_initial_batch(d, 3, grid=sf.PixelGrid(W, H))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    sf.estimate_initial_batch(d, 3, grid=sf.PixelGrid(W, H))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"initializer {W}x{H}: {ms:.3f} ms per 1e6 spots incl. the result copy to host ({n / ms * 1e3:.3g} spots/s)")
