"""Standalone GPU initializer throughput (sf_estimate_initial_device) on
HBM-resident spots: kernel time by CUDA events on the launching stream, and the achieved HBM
bandwidth (algorithmic bytes: 4 N per spot in, 4 P out) against MEASURED_PEAKS.json.

    python tools/init_bench.py [W] [count]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2106_02045_b200 as sf  # noqa: E402
from paper_2106_02045_b200.batch_engine import estimate_initial_device  # noqa: E402

W = H = int(sys.argv[1]) if len(sys.argv) > 1 else 15
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
im, _ = sf.simulate_batch_device(sf.SimConfig(width=W, height=H, count=n, seed=3))
d = im.reshape(n, W * H)
grid = sf.PixelGrid(W, H)
cfg = sf.FitConfig()
for _ in range(3):
    estimate_initial_device(d, grid, 3, cfg)
torch.cuda.synchronize()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record(st)
for _ in range(reps):
    estimate_initial_device(d, grid, 3, cfg)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
bytes_ = n * (4 * W * H + 4 * 3)
try:
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    peak = 7672.0
gbs = bytes_ / (ms * 1e-3) / 1e9
print(json.dumps({"grid": f"{W}x{H}", "spots": n, "ms": ms, "spots_per_s": n / ms * 1e3, "GBps": gbs,
                  "hbm_peak_GBps": peak, "frac": gbs / peak,
                  "note": "inputs 4N B/spot > L2 at 1e6 spots; result (count, 3) f32 stays on the device"}))
