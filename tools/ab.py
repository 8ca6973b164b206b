"""A/B harness: kernel-only fits/s (bench.py --profile) and a bitwise parity
spot-check for each library build given on the command line.

    python tools/ab.py default paper_2106_02045_b200/_lib/variants/*/libspotfit_b200.so
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PARITY = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2106_02045_b200 as sf
from oracle import lm, oracle_c
W = H = int(sys.argv[1]); model = int(sys.argv[2])
im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=20000, seed=77, model=min(model, 4)))
ini, amps = sf.estimate_initial_batch(im, 4 if model == 4 else 3)
if model == 5:  # explicit-5: (x, y, sigma) + the initializer's (alpha, beta)
    ini = np.ascontiguousarray(np.concatenate([ini, amps], axis=1).astype(np.float32))
r = sf.fit_batch(im, ini, engine={3: "implicit3", 4: "elliptical", 5: "explicit5"}[model])
ref = oracle_c.fit_batch(im.reshape(20000, -1), ini, W, H, lm.LMConfig.for_grid(W, H))
ok = all(np.array_equal(np.asarray(getattr(r, k)).view(np.uint8), np.asarray(ref[k]).view(np.uint8))
         for k in ("params", "alpha", "beta", "nchi2", "status", "iterations"))
print("PARITY", ok)
''' % ROOT


def run(lib, config="c2", count=1000000):
    env = dict(os.environ)
    if lib != "default":
        env["SPOTFIT_LIB"] = os.path.abspath(lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--profile", "--steps", "5", "--warmup", "3",
                          "--config", config, "--count", str(count)], capture_output=True, text=True, env=env)
    try:
        v = json.loads(out.stdout.strip().splitlines()[-1])["fits_per_s"]
    except Exception:
        v = None
        sys.stderr.write(out.stdout[-2000:] + out.stderr[-2000:])
    W, model = {"c2": (15, 3), "c1": (11, 3), "c3": (21, 4), "c4": (32, 3), "c2x": (15, 5)}[config]
    p = subprocess.run([sys.executable, "-c", PARITY, str(W), str(model)], capture_output=True, text=True, env=env)
    ok = "PARITY True" in p.stdout
    if not ok:
        sys.stderr.write(p.stdout[-1000:] + p.stderr[-1000:])
    return v, ok


if __name__ == "__main__":
    configs = os.environ.get("AB_CONFIGS", "c2").split(",")
    for lib in sys.argv[1:]:
        for c in configs:
            v, ok = run(lib, c)
            name = lib if lib == "default" else lib.split("/")[-2]
            print(f"AB {name:12s} {c}: {v/1e6 if v else float('nan'):8.2f} Mfits/s  parity={ok}", flush=True)
