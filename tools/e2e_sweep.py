"""e2e (public API, pinned host input and output buffers, as bench.py) fits/s vs the host pipeline's chunk cap
(SPOTFIT_CHUNK_MB), for f32 and u16 input.  One process per setting (the cap is read once)."""
import json
import os
import subprocess
import sys

CODE = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, %r)
import paper_2106_02045_b200 as sf
W = H = 15; n = 1_000_000
im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=n, seed=5))
ini, _ = sf.estimate_initial_batch(im, 3)
pin = torch.from_numpy(im.reshape(n, H, W)).pin_memory().numpy()
p16 = torch.from_numpy(im.reshape(n, H, W).astype(np.uint16)).pin_memory().numpy()
pini = torch.from_numpy(ini).pin_memory().numpy()
outs = sf.BatchResult(*[torch.empty(s, dtype=d).pin_memory().numpy() for s, d in [
    ((n, 3), torch.float32), (n, torch.float32), (n, torch.float32), (n, torch.float32),
    (n, torch.uint8), (n, torch.uint8)]])
out = {}
for name, x in (("f32", pin), ("u16", p16)):
    sf.fit_batch(x, pini, out=outs)
    t = time.perf_counter()
    for _ in range(5): sf.fit_batch(x, pini, out=outs)
    out[name] = 5 * n / (time.perf_counter() - t)
print("E2E", out)
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

for mb in sys.argv[1:] or ["64", "128", "256"]:
    env = dict(os.environ, SPOTFIT_CHUNK_MB=mb, SPOTFIT_CHUNK_MB16=mb)
    r = subprocess.run([sys.executable, "-c", CODE], capture_output=True, text=True, env=env)
    line = [l for l in r.stdout.splitlines() if l.startswith("E2E")]
    print(mb, "MB:", line[0] if line else r.stderr[-500:], flush=True)
