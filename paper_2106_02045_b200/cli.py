"""`spotfit` command line: simulate | fit | assess | bench.

    python -m paper_2106_02045_b200.cli simulate --size 15 --count 100000 --seed 1 --out spots.spb --truth truth.csv
    python -m paper_2106_02045_b200.cli fit --in spots.spb --out fits.csv
    python -m paper_2106_02045_b200.cli assess --fits fits.csv --truth truth.csv --report report.json
    python -m paper_2106_02045_b200.cli bench --sizes 9,15,21 --batches 10,1000,100000 --report bench.json

Exit codes: 0 ok, 2 invalid arguments, 3 I/O failure, 4 malformed SPB1 (with the byte offset).
`fit --engine implicit3` runs the CUDA fitter (the reference's CPU worker pool is replaced);
defaults are the paper's stop criteria (20 iterations, 1e-6, 1e-4).
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

EXIT_ARGS, EXIT_IO, EXIT_MALFORMED = 2, 3, 4


class CliError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _dump(obj, path):
    text = json.dumps(obj, sort_keys=True, indent=1)  # fixed lexical key order
    if path in (None, "-"):
        print(text)
    else:
        try:
            with open(path, "w") as f:
                f.write(text + "\n")
        except OSError as e:
            raise CliError(EXIT_IO, f"cannot write {path}: {e}")


def cmd_simulate(a):
    from .io_formats import write_spb1, write_truth_csv
    from .simulator import SimConfig, simulate_batch

    W = a.width or a.size
    H = a.height or a.size
    if W < 1 or H < 1 or W * H > 1024:
        raise CliError(EXIT_ARGS, f"grid {W}x{H} exceeds the 1024-pixel limit")
    if a.count < 0 or a.signal < 0 or a.background < 0 or not 0 < a.sigma_min <= a.sigma_max:
        raise CliError(EXIT_ARGS, "invalid simulation parameters")
    cfg = SimConfig(width=W, height=H, count=a.count, n_signal=a.signal, n_background=a.background,
                    sigma_range=(a.sigma_min, a.sigma_max), noise=not a.no_noise, rounding=not a.no_round,
                    seed=a.seed, model=4 if a.elliptical else 3)
    images, truth = simulate_batch(cfg)
    try:
        write_spb1(a.out, images)
        if a.truth:
            write_truth_csv(a.truth, truth)
    except OSError as e:
        raise CliError(EXIT_IO, str(e))
    return 0


def _load_spb1(path):
    from .io_formats import MalformedSPB1, read_spb1

    try:
        return read_spb1(path)
    except MalformedSPB1 as e:
        raise CliError(EXIT_MALFORMED, f"malformed SPB1 {path}: {e}")
    except OSError as e:
        raise CliError(EXIT_IO, f"cannot read {path}: {e}")


def _fit_config(a):
    from .solver import FitConfig

    try:
        return FitConfig(max_iterations=a.max_iter, max_error=a.max_error, min_delta=a.min_delta,
                         min_step=a.min_step)
    except ValueError as e:
        raise CliError(EXIT_ARGS, str(e))


def cmd_fit(a):
    from .batch_engine import fit_batch
    from .initializer import estimate_initial_batch
    from .io_formats import read_truth_csv, write_params_csv
    from .model import PixelGrid

    engines = {"implicit3": 3, "elliptical": 4, "explicit5": 5}
    if a.engine not in engines:
        raise CliError(EXIT_ARGS, f"unknown engine {a.engine!r} (implicit3 | explicit5 | elliptical)")
    images, W, H = _load_spb1(a.inp)
    cfg = _fit_config(a)
    P = engines[a.engine]
    grid = PixelGrid(W, H)
    count = images.shape[0]
    flat = np.ascontiguousarray(images).reshape(count, W * H)
    t0 = time.perf_counter()
    if a.inits in (None, "auto"):
        if count == 0:
            inits = np.zeros((0, P), np.float32)
        elif P == 5:  # explicit5 also starts from the initializer's alpha, beta
            ini, amps = estimate_initial_batch(flat, 3, cfg, grid=grid)
            inits = np.concatenate([ini, amps], axis=1)
        else:
            inits = estimate_initial_batch(flat, P, cfg, grid=grid)[0]
    else:
        try:
            t = read_truth_csv(a.inits)  # x, y, sigma[, sigma_y], alpha, beta
            inits = np.concatenate([t[:, :3], t[:, -2:]], axis=1) if P == 5 else t[:, :P]
        except (OSError, ValueError) as e:
            raise CliError(EXIT_IO, f"cannot read inits {a.inits}: {e}")
        if len(inits) != count:
            raise CliError(EXIT_ARGS, f"inits has {len(inits)} rows for {count} images")
    t1 = time.perf_counter()
    devices = [int(d) for d in a.devices.split(",")] if a.devices else None
    res = fit_batch(flat, inits, config=cfg, engine=a.engine, grid=grid, devices=devices)
    t2 = time.perf_counter()
    try:
        write_params_csv(a.out, res, flags=a.flags)
    except OSError as e:
        raise CliError(EXIT_IO, str(e))
    fit_s = t2 - t1
    sys.stderr.write(f"spotfit: {count} fits of {W}x{H} in {fit_s * 1e3:.1f} ms "
                     f"({count / fit_s if fit_s > 0 else 0:.3g} fits/s; init {1e3 * (t1 - t0):.1f} ms)\n")
    return 0


def cmd_assess(a):
    from .assess import accuracy, expected_error_ratio, iteration_stats
    from .io_formats import read_params_csv, read_truth_csv

    try:
        fits = read_params_csv(a.fits)
        truth = read_truth_csv(a.truth)
    except (OSError, ValueError) as e:
        raise CliError(EXIT_IO, f"cannot read inputs: {e}")
    if len(truth) != len(fits["alpha"]):
        raise CliError(EXIT_ARGS, "fits and truth differ in length")
    stats = accuracy(fits["params"], fits["stop"], truth)
    status = fits["stop"] | fits["flags"] if "flags" in fits else fits["stop"]
    its = iteration_stats(status, fits["iterations"], max(int(a.max_iter), int(fits["iterations"].max(initial=0))))
    if "flags" not in fits:  # the SPEC header carries the StopReason name only
        its["no_improvement"] = None
        its["invalid_input"] = None
        sys.stderr.write("spotfit assess: no flags column (fit --flags): no-improvement / invalid counts unavailable\n")
    report = {"accuracy": stats.as_dict(), "iterations": its}
    if a.signal:
        report["expected_error_ratio"] = expected_error_ratio(stats, a.signal)
    _dump(report, a.report)
    return 0


REPEATS = {10: 200, 100: 20, 1000: 10, 10000: 1}  # PAPER.md Results: "run 200x, 20x, 10x and once"


def bench_plan(sizes: str, batches: str, repeats: str = ""):
    """SPEC.md:475-478 BenchPlan -> [(S, batch, repeats)]: sizes "4-32" (a range) or a comma list,
    batch sizes with the paper's repeat counts unless given."""
    if "-" in sizes:
        lo, hi = (int(v) for v in sizes.split("-"))
        S = list(range(lo, hi + 1))
    else:
        S = [int(v) for v in sizes.split(",")]
    B = [int(v) for v in batches.split(",")]
    R = [int(v) for v in repeats.split(",")] if repeats else [REPEATS.get(b, max(1, 2000 // b)) for b in B]
    if any(s < 1 or s * s > 1024 for s in S) or any(b < 1 for b in B) or len(R) != len(B) or min(R) < 1:
        raise CliError(EXIT_ARGS, "sizes must satisfy S*S <= 1024; batches and repeats >= 1, one repeat per batch")
    return [(s, b, r) for s in S for b, r in zip(B, R)]


def cmd_bench(a):
    """SPEC.md:471-512 run_bench: per (S, batch) mean wall time of fit_batch from host memory
    (marshaling + fit + result collection), inits excluded, after a warm-up call; monotonic clock;
    timings under 5 clock ticks are flagged."""
    from .batch_engine import fit_batch
    from .initializer import estimate_initial_batch
    from .model import PixelGrid
    from .simulator import SimConfig, simulate_batch

    plan = bench_plan(a.sizes, a.batches, a.repeats)
    tick = time.get_clock_info("perf_counter").resolution
    entries = []
    for S, B, reps in plan:
        grid = PixelGrid(S, S)
        im, _ = simulate_batch(SimConfig(width=S, height=S, count=B, seed=S * 1000 + B, n_signal=a.signal,
                                         n_background=a.background))
        flat = im.reshape(B, S * S)
        ini, amps = estimate_initial_batch(flat, 3, grid=grid)
        if a.engine == "explicit5":  # (x, y, sigma) + the initializer's (alpha, beta)
            ini = np.ascontiguousarray(np.concatenate([ini, amps], axis=1), dtype=np.float32)
        fit_batch(flat, ini, grid=grid, engine=a.engine)  # warm-up
        t0 = time.perf_counter()
        for _ in range(reps):
            fit_batch(flat, ini, grid=grid, engine=a.engine)
        dt = (time.perf_counter() - t0) / reps
        entries.append({"size": S, "batch": B, "repeats": reps, "seconds_per_call": dt, "fits_per_s": B / dt,
                        "pixels_per_s": B * S * S / dt, "under_resolved": dt < 5 * tick})
    import torch

    _dump({"machine": torch.cuda.get_device_name(0), "engine": a.engine + "/cuda", "entries": entries}, a.report)
    if a.csv:
        with open(a.csv, "w") as f:
            f.write("size,batch,repeats,seconds_per_call,fits_per_s,pixels_per_s\n")
            for e in entries:
                f.write(f"{e['size']},{e['batch']},{e['repeats']},{e['seconds_per_call']!r},{e['fits_per_s']!r},"
                        f"{e['pixels_per_s']!r}\n")
    return 0


def build_parser():
    p = argparse.ArgumentParser(prog="spotfit", description=__doc__.split("\n")[0])
    sub = p.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("simulate")
    s.add_argument("--size", type=int, default=9)
    s.add_argument("--width", type=int, default=0)
    s.add_argument("--height", type=int, default=0)
    s.add_argument("--count", type=int, default=1000)
    s.add_argument("--signal", type=float, default=400.0)
    s.add_argument("--background", type=float, default=40.0)
    s.add_argument("--sigma-min", type=float, default=1.0)
    s.add_argument("--sigma-max", type=float, default=2.0)
    s.add_argument("--no-noise", action="store_true")
    s.add_argument("--no-round", action="store_true")
    s.add_argument("--elliptical", action="store_true")
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--out", required=True)
    s.add_argument("--truth")
    f = sub.add_parser("fit")
    f.add_argument("--in", dest="inp", required=True)
    f.add_argument("--out", required=True)
    f.add_argument("--engine", default="implicit3")
    f.add_argument("--max-iter", type=int, default=20)
    f.add_argument("--min-delta", type=float, default=1e-6)
    f.add_argument("--min-step", type=float, default=1e-4)
    f.add_argument("--max-error", type=float, default=0.0)
    f.add_argument("--workers", type=int, default=0, help="accepted for compatibility (GPU engine)")
    f.add_argument("--devices", default="")
    f.add_argument("--inits", default="auto")
    f.add_argument("--flags", action="store_true",
                   help="append a flags column (status & 0xf8: 64 InvalidInput, 128 no-improvement) for assess")
    a = sub.add_parser("assess")
    a.add_argument("--fits", required=True)
    a.add_argument("--truth", required=True)
    a.add_argument("--report")
    a.add_argument("--signal", type=float, default=0.0)
    a.add_argument("--max-iter", type=int, default=20, help="histogram range (the fit's --max-iter)")
    b = sub.add_parser("bench")
    b.add_argument("--sizes", default="4-32", help="range lo-hi or a comma list (SPEC.md:475: S = 4..32)")
    b.add_argument("--batches", default="10,100,1000,10000")
    b.add_argument("--repeats", default="", help="per batch size (default 200, 20, 10, 1 as the paper)")
    b.add_argument("--csv", default="", help="optional CSV table, one row per (S, batch)")
    b.add_argument("--signal", type=float, default=400.0)
    b.add_argument("--background", type=float, default=40.0)
    b.add_argument("--engine", default="implicit3")
    b.add_argument("--report")
    return p


def main(argv=None) -> int:
    p = build_parser()
    try:
        a = p.parse_args(argv)
    except SystemExit as e:
        return EXIT_ARGS if e.code not in (0, None) else 0
    try:
        return {"simulate": cmd_simulate, "fit": cmd_fit, "assess": cmd_assess, "bench": cmd_bench}[a.cmd](a)
    except CliError as e:
        sys.stderr.write(f"spotfit: {e}\n")
        return e.code


def entry():
    sys.exit(main())


if __name__ == "__main__":
    entry()
