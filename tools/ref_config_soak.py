"""CPU soak pinning the C oracle to the reference itself over the configuration space:
the LM loop oracle/lm.py over the UNMODIFIED reference spotfit.model (baseline/_ref) vs
oracle/spotfit_oracle.c, on tools/config_soak.make_case cases (symmetric model: the
reference has no elliptical or explicit-5 model code).  No GPU needed (host simulator).

    python tools/ref_config_soak.py [rounds] [seed]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import config_soak  # noqa: E402
from oracle import lm, oracle_c  # noqa: E402

if __name__ == "__main__":
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 45)
    _, kind = lm.model_backend("reference")
    assert kind == "reference", "reference spotfit not installed under baseline/_ref"
    t0, fits, fails = time.time(), 0, 0
    for r in range(rounds):
        c = config_soak.make_case(rng, models=(3,), counts=(60, 200))
        ref = lm.fit_batch_parallel(c["im"], c["ini"], c["W"], c["H"], c["ocfg"], backend="reference")
        got = oracle_c.fit_batch(c["im"], c["ini"], c["W"], c["H"], c["ocfg"])
        bad = [k for k in config_soak.FIELDS
               if not np.array_equal(np.asarray(got[k]).view(np.uint8), np.asarray(ref[k]).view(np.uint8))]
        stops = np.bincount(np.asarray(got["status"]) & 7, minlength=5)
        print(f"round {r:3d}: {c['W']:2d}x{c['H']:2d} n={c['count']:3d} it<={c['kw']['max_iterations']:2d} "
              f"stops={stops.tolist()} {'ok' if not bad else 'MISMATCH ' + ','.join(bad)}", flush=True)
        fits += c["count"]
        fails += bool(bad)
    print(f"REF_CONFIG_SOAK rounds={rounds} fits={fits} mismatching_rounds={fails} ({time.time() - t0:.0f} s)")
