"""Statistical acceptance at scale (SPEC.md ACCEPTANCE CRITERIA 1-5; Table 1 and Fig. 8,
PAPER.md:262-284) on the GPU: simulate -> initialise -> fit -> assess, 1e6 spots per setting.

  1. Table 1, 400:40, S = 9: position median/mean/std and sigma median within +-10% of
     0.0464 / 0.0550 / 0.0418 and 0.0420.
  2. Table 1, 1600:40: position median/mean within +-10% of 0.0228 / 0.0270, sigma median of 0.0203.
  3. Shot-noise ratio at 1600:0: mean position error / (1/sqrt(1600)) in [1.0, 1.2].
  4. Iterations at 1600:40: implicit3 histogram mode in {4, 5}; mean(implicit3) < mean(explicit5)
     on the same inputs with identical initial estimates.
  5. Stops at 1600:40: MinDelta family dominates; no-improvement 15% +- 10 points; MinStep < 2%;
     MaxIterations <= 0.1%.

Everything runs on the device (simulator, initializer, fit); assess.py computes the statistics.

    python tools/acceptance.py [--count 1000000] [--out profiles/r02_acceptance.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TABLE1 = {  # PAPER.md:269-273, Fit2DGaussian rows: position median/mean/std, sigma median/mean/std
    "400:40": (0.0464, 0.0550, 0.0418, 0.0420, 0.0506, 0.0396),
    "1600:40": (0.0228, 0.0270, 0.0205, 0.0203, 0.0244, 0.0190),
    "1600:0": (0.0228, 0.0269, 0.0203, 0.0198, 0.0238, 0.0186),
}


def within(got, want, rel=0.10):
    return bool(abs(got - want) <= rel * want)


def run_setting(sf, S, signal, background, count, seed, engines=("implicit3",)):
    import torch

    from paper_2106_02045_b200.assess import accuracy, iteration_stats
    from paper_2106_02045_b200.batch_engine import estimate_initial_device

    grid = sf.PixelGrid(S, S)
    cfg = sf.SimConfig(width=S, height=S, count=count, n_signal=signal, n_background=background, seed=seed)
    t0 = time.perf_counter()
    im, truth = sf.simulate_batch_device(cfg)
    flat = im.reshape(count, S * S)
    ini, am = estimate_initial_device(flat, grid, 3, sf.FitConfig(), amps=True)
    torch.cuda.synchronize()
    truth_np = truth.cpu().numpy()
    out = {"spots": count, "S": S, "signal": signal, "background": background, "seed": seed}
    for eng in engines:
        inits = ini if eng == "implicit3" else torch.cat([ini, am], dim=1).contiguous()
        t1 = time.perf_counter()
        r = sf.fit_batch(flat, inits, engine=eng, grid=grid)
        dt = time.perf_counter() - t1
        acc = accuracy(r.params[:, :3], r.status, truth_np)
        it = iteration_stats(r.status, r.iterations, 20)
        n = it["n_fits"]
        stops = it["stop_reasons"]
        out[eng] = {
            "accuracy": acc.as_dict(),
            "iterations": {"mode": it["mode"], "mean": it["mean"], "histogram": it["histogram"]},
            "stops": stops,
            "frac": {
                "min_delta_family": (stops["MinDelta"] + stops["MaxError"]) / n,
                "no_improvement": it["no_improvement"] / n,
                "min_step": stops["MinStep"] / n,
                "max_iterations": stops["MaxIterations"] / n,
                "not_converged": stops["NotConverged"] / n,
            },
            "sigma_negated": int((r.params[:, 2] < 0).sum()),
            "fit_s": dt,
        }
    out["wall_s"] = time.perf_counter() - t0
    return out


def main(argv=None):
    import paper_2106_02045_b200 as sf

    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=1_000_000)
    ap.add_argument("--size", type=int, default=9)
    ap.add_argument("--out", default="")
    a = ap.parse_args(argv)
    res = {"count_per_setting": a.count, "S": a.size, "table1": TABLE1}
    res["400:40"] = run_setting(sf, a.size, 400.0, 40.0, a.count, 4040)
    res["1600:40"] = run_setting(sf, a.size, 1600.0, 40.0, a.count, 16040, engines=("implicit3", "explicit5"))
    res["1600:0"] = run_setting(sf, a.size, 1600.0, 0.0, a.count, 16000)
    crit = {}
    for key, rows in (("400:40", (0, 1, 2, 3)), ("1600:40", (0, 1, 3))):
        acc = res[key]["implicit3"]["accuracy"]
        got = (acc["position_median"], acc["position_mean"], acc["position_std"], acc["sigma_median"],
               acc["sigma_mean"], acc["sigma_std"])
        crit[f"table1_{key}"] = {
            "pass": all(within(got[i], TABLE1[key][i]) for i in rows),
            "got": got, "paper": TABLE1[key],
            "checked": [("pos_median", "pos_mean", "pos_std", "sigma_median", "sigma_mean", "sigma_std")[i] for i in rows],
        }
    ratio = res["1600:0"]["implicit3"]["accuracy"]["position_mean"] * np.sqrt(1600.0)
    crit["shot_noise_ratio_1600_0"] = {"pass": bool(1.0 <= ratio <= 1.2), "value": float(ratio), "range": [1.0, 1.2]}
    i3, e5 = res["1600:40"]["implicit3"], res["1600:40"]["explicit5"]
    crit["iterations_1600_40"] = {
        "pass": i3["iterations"]["mode"] in (4, 5) and i3["iterations"]["mean"] < e5["iterations"]["mean"],
        "implicit3_mode": i3["iterations"]["mode"], "implicit3_mean": i3["iterations"]["mean"],
        "explicit5_mode": e5["iterations"]["mode"], "explicit5_mean": e5["iterations"]["mean"],
    }
    f = i3["frac"]
    crit["stops_1600_40"] = {
        "pass": bool(f["min_delta_family"] > 0.5 and abs(f["no_improvement"] - 0.15) <= 0.10 and f["min_step"] < 0.02
                     and f["max_iterations"] <= 0.001),
        **f,
    }
    res["criteria"] = crit
    res["all_pass"] = all(c["pass"] for c in crit.values())
    text = json.dumps(res, indent=1)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text + "\n")
    print(json.dumps({k: v["pass"] for k, v in crit.items()}), "all_pass", res["all_pass"])
    print(json.dumps(crit, indent=1))


if __name__ == "__main__":
    main()
