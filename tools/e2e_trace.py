"""Per-chunk device timeline of the host pipeline (SPOTFIT_TRACE=1), f32 and u16 input.

    SPOTFIT_TRACE=1 python tools/e2e_trace.py [count]

Prints per chunk: H2D window, the ready -> fit-done window, and a summary of
how much of the wall span a fit kernel was running (union of fit windows)."""
import os
import subprocess
import sys

CHILD = r'''
import sys, time, numpy as np
sys.path.insert(0, %r)
import paper_2106_02045_b200 as sf
count = int(sys.argv[1]); u16 = sys.argv[2] == "u16"
im, _ = sf.simulate_batch(sf.SimConfig(width=15, height=15, count=count, seed=5))
ini, _ = sf.estimate_initial_batch(im, 3)
import torch
imgs = torch.from_numpy(im.astype(np.uint16) if u16 else im).pin_memory().numpy()
inis = torch.from_numpy(ini).pin_memory().numpy()
for _ in range(2):
    sf.fit_batch(imgs, inis)
sys.stderr.write("RUN\n")
t = time.perf_counter(); sf.fit_batch(imgs, inis); dt = time.perf_counter() - t
print("WALL", dt, count / dt)
'''


def analyse(lines):
    rows = [list(map(float, l.split()[1:])) for l in lines]
    fit = sorted((r[2], r[3]) for r in rows)
    union, cur = 0.0, None
    for a, b in fit:
        if cur is None or a > cur[1]:
            if cur:
                union += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    union += cur[1] - cur[0]
    end = max(r[4] for r in rows)
    for i, r in enumerate(rows):
        print(f"chunk {i:2d}: h2d {r[0]:7.3f}-{r[1]:7.3f}  ready {r[2]:7.3f}  fit-done {r[3]:7.3f} ({r[3]-r[2]:6.3f})  d2h {r[4]:7.3f}")
    print(f"span {end:.3f} ms, first ready {rows[0][2]:.3f}, fit union {union:.3f} ms, "
          f"gaps {rows[-1][3] - rows[0][2] - union:.3f} ms, last d2h {end - rows[-1][3]:.3f}")


if __name__ == "__main__":
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    count = sys.argv[1] if len(sys.argv) > 1 else "1000000"
    env = dict(os.environ, SPOTFIT_TRACE="1")
    for kind in ("f32", "u16"):
        p = subprocess.run([sys.executable, "-c", CHILD % root, count, kind], capture_output=True, text=True, env=env)
        err = p.stderr.split("RUN\n")[-1]
        tr = [l for l in err.splitlines() if l.startswith("TRACE")]
        print(f"== {kind}: {p.stdout.strip()}")
        if tr:
            analyse(tr)
        else:
            print(p.stderr[-2000:])
