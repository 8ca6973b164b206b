"""bench.py -- headline benchmark: 2D Gaussian fits/s (15x15 px, symmetric,
implicit alpha/beta) on N B200s vs the reference CPU fitter.

Workload (BASELINE.json configs[1]): 1e6 synthetic spots per GPU
(weak scaling), 15x15 px, 400:40 counts, Poisson-like noise (simulator seed
2021, global spot index = device * 1e6 + i), inits from the untimed GPU
initializer, exactly as PAPER.md:210-212 times the fit.  A step = one full LM
fit of the whole batch on every GPU.

  value      -- fits/s with inputs resident in HBM (sf_fit_batch_device per GPU,
                CUDA events on each launching stream, max over GPUs); 900 MB of
                input per GPU > 126 MB L2, so no L2 flush is needed between steps.
  e2e        -- the drop-in call fit_batch(images) (inits=None: the fit kernel's
                fused initializer) from pinned host memory, H2D + kernel + D2H
                inside the timed region; e2e_variants: with inits (the paper's
                span), pageable numpy, u16 counts.
  per_config -- BASELINE configs 1, 3 and 4 (c4 at its full 1e7 spots) and the
                explicit-5 baseline on one GPU: kernel fits/s, roofline fraction
                and a bitwise parity sample.
  c5         -- BASELINE configs[4]: 1e8 15x15 spots (total, strong scaling) from
                pinned host memory through fit_batch(devices=all), with a parity
                sample around the shard boundaries, plus the real-time mode
                (50 spots per frame at 1 kHz).
  --impl reference -- the reference CPU fitter (the unmodified reference
                spotfit.model from baseline/_ref under the restated LM loop) on all
                host cores, bounded sample per step; inputs from oracle/simulator.py.

Multi-GPU: ``python bench.py --gpus N`` drives N devices from one process (one
host thread per device inside sf_fit_batch; per-device streams for the kernel
leg); under torchrun each rank drives its LOCAL_RANK device and gloo carries the
barrier and the max-over-ranks reduction (no collective on the data path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (W, H, spots per GPU, model)
    "c2": (15, 15, 1_000_000, 3),
    "c1": (11, 11, 10_000, 3),
    "c3": (21, 21, 1_000_000, 4),
    "c4": (32, 32, 10_000_000, 3),
    "c2x": (15, 15, 1_000_000, 5),  # explicit 5-parameter baseline on the C2 workload
}
SEED = 2021
METRIC = "2D Gaussian fits/sec (15x15 px) at 1/2/4/8 B200 vs CPU ref; % FP32/SFU roofline"
# algorithmic work per pixel-evaluation: G-eval 67 ops (45 FP32 + 22 reduction adds),
# T-eval 18 ops (14 + 4); one exp each.  Elliptical G-eval: 58 + 30.
OPS_G = {3: 67, 4: 88, 5: 60}  # explicit-5: 39 FP32 + 21 reduction adds per pixel-evaluation (G = T)
OPS_T = {3: 18, 4: 18, 5: 60}
MODEL_NAME = {3: "symmetric", 4: "elliptical", 5: "explicit-5"}
ENGINE = {3: "implicit3", 4: "elliptical", 5: "explicit5"}
FIELDS = ("params", "alpha", "beta", "nchi2", "status", "iterations")


def host_info() -> dict:
    """CPU model and numpy's float32 SIMD dispatch (the reference's exp is numpy's SIMD kernel)."""
    cpu = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    cpu = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    simd = []
    try:
        from numpy._core._multiarray_umath import __cpu_features__ as feats  # numpy >= 2
    except ImportError:  # pragma: no cover
        try:
            from numpy.core._multiarray_umath import __cpu_features__ as feats
        except ImportError:
            feats = {}
    for k in ("AVX512_SPR", "AVX512_ICL", "AVX512_SKX", "AVX512F", "AVX2", "FMA3"):
        if feats.get(k):
            simd.append(k)
    return {"cpu": cpu, "numpy": np.__version__, "simd": simd[:3]}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region.  nvidia-smi takes a few
    hundred ms to start, longer than a 20-step timed region, so the sampler is started (and its first
    row awaited) before the warm-up; rows carry the host time they arrived, and the summary keeps the
    rows inside the timed window (+- one sampling period), else the rows bracketing it."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    PERIOD_S = 0.1

    def __init__(self, gpus):
        self.gpus, self.rows, self.proc = sorted(set(gpus)), [], None
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", ",".join(str(g) for g in self.gpus),
                                          f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                                          str(int(self.PERIOD_S * 1000))],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.monotonic() + 3.0
            while not self.rows and time.monotonic() < deadline:  # the sampler is live before timing starts
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append((time.monotonic(), parts))

    def begin(self):
        self.t0 = time.monotonic()

    def end(self):
        self.t1 = time.monotonic()
        # one more sampling period so the rows covering the end of the window arrive
        time.sleep(1.5 * self.PERIOD_S)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = self.rows
        how = "in the timed window"
        if self.t0 is not None and self.t1 is not None:
            inside = [r for t, r in rows if self.t0 - self.PERIOD_S <= t <= self.t1 + self.PERIOD_S]
            if not inside:  # the rows on either side of the window
                before = [r for t, r in rows if t < self.t0][-1:]
                after = [r for t, r in rows if t > self.t1][:1]
                inside = before + after
                how = "bracketing the timed window"
            rows = inside
        else:
            rows = [r for _, r in rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "sampled": how,
                "window_s": None if self.t0 is None else self.t1 - self.t0}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def workload_config(args, n_gpus: int) -> dict:
    """The `config` object of the bench line -- identical in both arms (the reference arm times a
    bounded sample of this same workload and says so in cpu_baseline.sample)."""
    W, H, count, model = CONFIGS[args.config]
    count = args.count or count
    return {"workload": f"{args.config}: {count} {MODEL_NAME[model]} spots/GPU, {W}x{H} px, max 20 LM iterations, "
                        f"simulator seed {SEED}", "spots_per_gpu": count, "W": W, "H": H, "model": model,
            "parallelism": f"independent shards x{n_gpus}",
            "l2": f"inputs {count * W * H * 4 / 1e6:.0f} MB/GPU > 126 MB L2 (no flush needed)"}


# ----------------------------------------------------------------------------- reference arm
def cpu_reference(W, H, model, images, inits, sample, workers):
    """The reference CPU fitter on `sample` spots, all host cores -> (fits/s, seconds, kind).

    Arithmetic: the unmodified reference spotfit.model (pkg/src/spotfit/model.py)
    pip-installed into baseline/_ref -- kind "reference" -- driven by the
    restated LM loop oracle/lm.py (the reference ships no solver code); the
    elliptical model has no reference code, so it runs on oracle/model_np.py
    (kind "port")."""
    from oracle import lm

    backend = "auto" if model in (3, 5) else "port"
    _, kind = lm.model_backend(backend)
    cfg = lm.LMConfig.for_grid(W, H)
    t0 = time.perf_counter()
    lm.fit_batch_parallel(images[:sample], inits[:sample], W, H, cfg, workers=workers, backend=backend)
    dt = time.perf_counter() - t0
    return sample / dt, dt, kind


def cpu_c_port(W, H, images, inits, sample, threads):
    from oracle import lm, oracle_c

    cfg = lm.LMConfig.for_grid(W, H)
    t0 = time.perf_counter()
    oracle_c.fit_batch(images[:sample], inits[:sample], W, H, cfg, threads=threads)
    return sample / (time.perf_counter() - t0)


def reference_inputs(W, H, model, sample):
    """The first `sample` spots of the GPU arm's workload (seed SEED, indices 0..sample-1) and their
    inits, built by the oracle's restatements only (no product library in this process)."""
    from oracle import initializer as oinit
    from oracle import simulator as osim

    sim_model = 4 if model == 4 else 3
    images, _ = osim.simulate_batch(W, H, sample, SEED, model=sim_model)
    images = images.reshape(sample, W * H)
    inits, amps = oinit.estimate_initial_batch_np(images, W, H, 0.3, float(max(W, H)), min(model, 4))
    if model == 5:
        inits = np.ascontiguousarray(np.concatenate([inits, amps], axis=1).astype(np.float32))
    return images, inits


def run_reference(args):
    rank, world, _ = dist_env()
    W, H, count, model = CONFIGS[args.config]
    if rank != 0:
        return 0
    cores = len(os.sched_getaffinity(0))
    sample = args.ref_sample or max(4000, 1500 * cores)
    images, inits = reference_inputs(W, H, model, sample)
    for _ in range(args.warmup):
        cpu_reference(W, H, model, images, inits, min(sample, 64 * cores), cores)
    times = []
    kind = "port"
    for _ in range(args.steps):
        _, dt, kind = cpu_reference(W, H, model, images, inits, sample, cores)
        times.append(dt)
    total = float(np.sum(times))
    value = sample * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "fits/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (per-pixel) / f64 (sums)",
        "data": "synthetic (SPEC.md:316-368 simulator restated in oracle/simulator.py, 400:40 counts, seeded)",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "fits/s", "cores": cores, "kind": kind, "host": host_info(),
                         "sample": f"spots 0..{sample - 1} of the {W}x{H} workload (the GPU arm's first {sample} "
                                   f"spots) per step, {args.steps} steps; arithmetic: reference spotfit.model from "
                                   "baseline/_ref, LM loop oracle/lm.py; inits oracle/initializer.py"},
        "e2e": {"value": value, "unit": "fits/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "inputs": "oracle/simulator.py + oracle/initializer.py (the product library is not loaded in this arm)",
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- our arm: helpers
def parity(got, images, inits, W, H):
    """Bitwise comparison of GPU results (dict of arrays, one row per sampled spot) with the C
    oracle fitting the same images from the same inits."""
    from oracle import lm, oracle_c

    ref = oracle_c.fit_batch(np.ascontiguousarray(images), np.ascontiguousarray(inits), W, H,
                             lm.LMConfig.for_grid(W, H))
    n = len(images)
    same = np.ones(n, bool)
    for k in FIELDS:
        a, b = np.asarray(got[k]), np.asarray(ref[k])
        eq = (a.view(np.uint8).reshape(n, -1) == b.view(np.uint8).reshape(n, -1)).all(axis=1)
        if a.dtype.kind == "f":  # NaN results (InvalidInput / singular) match any NaN
            eq |= (np.isnan(a.astype(np.float64)) & np.isnan(b.astype(np.float64))).reshape(n, -1).all(axis=1)
        same &= eq
    return {"sample": int(n), "bitwise_identical_frac": float(same.mean()),
            "state_identical_frac": float((np.asarray(got["status"]) == ref["status"]).mean()),
            "checker": "oracle/spotfit_oracle.c (pinned to reference model.py fixtures)"}


def roofline_of(model, N, count, evs, launch_s, sms, sm_max_mhz):
    n_g, n_t, n_k = evs
    ops = N * (OPS_G[model] * n_g + OPS_T[model] * n_t)
    fp32_peak = sms * 128 * sm_max_mhz * 1e6
    return {"achieved": ops / launch_s / 1e12, "peak": fp32_peak / 1e12, "unit": "TOP/s",
            "frac": ops / launch_s / fp32_peak, "ops_per_fit": ops / count,
            "evals_per_fit": {"n_G": n_g / count, "n_T": n_t / count, "kernel": n_k / count}}


class Devices:
    """The GPUs this process drives: [LOCAL_RANK] under torchrun, else --devices / range(--gpus)."""

    def __init__(self, args):
        import torch

        self.rank, self.world, self.local = dist_env()
        ndev = torch.cuda.device_count()
        if self.world > 1:
            self.ids = [self.local % ndev]
        elif args.devices:
            self.ids = [int(x) for x in args.devices.split(",")]
        else:
            if args.gpus > ndev:
                raise SystemExit(f"--gpus {args.gpus} but only {ndev} CUDA device(s) are visible")
            self.ids = list(range(args.gpus))
        if any(d >= ndev for d in self.ids):
            raise SystemExit(f"device ids {self.ids} out of range ({ndev} visible)")
        torch.cuda.set_device(self.ids[0])
        self.n_gpus = self.world * len(self.ids)  # GPUs (or emulated device slots) in the whole job
        if self.world > 1:
            import torch.distributed as dist

            # plumbing only (barrier + max over ranks): the fits exchange no data
            dist.init_process_group("gloo")

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier()

    def _reduce(self, x: float, op) -> float:
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x: float) -> float:
        import torch.distributed as dist

        return self._reduce(x, dist.ReduceOp.MAX)

    def sum(self, x: float) -> float:
        import torch.distributed as dist

        return self._reduce(x, dist.ReduceOp.SUM)

    def close(self):
        if self.world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


class _Single:
    """Devices stand-in for single-device legs."""

    world = 1

    def barrier(self):
        pass

    def max(self, x):
        return x


def device_batch(sf, dev, W, H, count, model, first_index, host=True):
    """Synthetic spots on device `dev` (+ the host copy when host=True: the C2 inputs come from the
    host generator, bit-identical to the reference arm's oracle/simulator.py) and the standalone
    GPU initializer's inits (untimed)."""
    import torch

    sim_model = 4 if model == 4 else 3
    cfgsim = sf.SimConfig(width=W, height=H, count=count, seed=SEED, model=sim_model)
    with torch.cuda.device(dev):
        if host:
            images, _ = sf.simulate_batch(cfgsim, first_index=first_index)
            images = images.reshape(count, W * H)
            d_img = torch.from_numpy(images).to(dev)
        else:
            images = None
            d_img, _ = sf.simulate_batch_device(cfgsim, first_index=first_index, device=dev)
            d_img = d_img.reshape(count, W * H)
        grid = sf.PixelGrid(W, H)
        if model == 5:
            ini, am = sf.batch_engine.estimate_initial_device(d_img, grid, 3, sf.FitConfig(), amps=True)
            d_ini = torch.cat([ini, am], dim=1).contiguous()
        else:
            d_ini = sf.batch_engine.estimate_initial_device(d_img, grid, model, sf.FitConfig())
        torch.cuda.synchronize(dev)
    return images, d_img, d_ini


class KernelLeg:
    """sf_fit_batch_device on HBM-resident inputs of one device: output buffers, stream, counters."""

    def __init__(self, sf, dev, W, H, count, model, d_img, d_ini):
        import ctypes

        import torch

        self.sf, self.dev, self.W, self.H, self.count, self.model = sf, dev, W, H, count, model
        self.d_img, self.d_ini = d_img, d_ini
        with torch.cuda.device(dev):
            self.d_par = torch.empty((count, model), dtype=torch.float32, device=dev)
            self.d_f = torch.empty((3, count), dtype=torch.float32, device=dev)
            self.d_u8 = torch.empty((2, count), dtype=torch.uint8, device=dev)
            self.d_ev = torch.zeros(3, dtype=torch.int64, device=dev)
            self.stream = torch.cuda.Stream(dev)
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e1 = torch.cuda.Event(enable_timing=True)
        self.ccfg = sf.FitConfig().to_c(sf.PixelGrid(W, H), model)
        self.byref = ctypes.byref

    def launch(self):
        L = self.sf._lib.lib()
        self.sf._lib.check(L.sf_fit_batch_device(
            self.d_img.data_ptr(), self.W, self.H, self.count, self.d_ini.data_ptr(), self.byref(self.ccfg),
            self.d_par.data_ptr(), self.d_f[0].data_ptr(), self.d_f[1].data_ptr(), self.d_f[2].data_ptr(),
            self.d_u8[0].data_ptr(), self.d_u8[1].data_ptr(), self.d_ev.data_ptr(), self.stream.cuda_stream))

    def results(self, idx):
        import torch

        ti = torch.from_numpy(np.asarray(idx, np.int64)).to(self.dev)
        par = self.d_par.index_select(0, ti).cpu().numpy()
        f = self.d_f.index_select(1, ti).cpu().numpy()
        u8 = self.d_u8.index_select(1, ti).cpu().numpy()
        return {"params": par, "alpha": f[0], "beta": f[1], "nchi2": f[2], "status": u8[0], "iterations": u8[1]}


def initializer_leg(sf, dev, d_img, W, H, count, model, reps=10):
    """The standalone GPU initializer (sf_estimate_initial_device, sf_init.cu) on the headline's
    HBM-resident batch (> L2), CUDA events on the launching stream.  Not part of `value` (PAPER.md:212
    times the fit from given inits); it runs in front of the fit for inits=None batches above the
    fused-initializer size.  Bytes: 4N in + 4P out per spot."""
    import torch

    grid, cfg, P = sf.PixelGrid(W, H), sf.FitConfig(), min(model, 4) if model != 5 else 3
    with torch.cuda.device(dev):
        for _ in range(3):
            sf.batch_engine.estimate_initial_device(d_img, grid, P, cfg)
        st = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(st)
        for _ in range(reps):
            sf.batch_engine.estimate_initial_device(d_img, grid, P, cfg)
        e1.record(st)
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / reps
    gbs = count * (4 * W * H + 4 * P) / (ms * 1e-3) / 1e9
    peak = load_peaks().get("hbm_gbs")
    return {"ms_per_launch": ms, "spots_per_s": count / (ms * 1e-3), "achieved_GBps": gbs, "peak_GBps": peak,
            "frac": gbs / peak if peak else None, "launches": reps, "bytes_per_spot": 4 * W * H + 4 * P,
            "note": "standalone initializer on the headline batch (> L2), untimed by `value`"}


def time_legs(legs, steps, warmup, devs, clock=None):
    """Launch every leg `steps` times (all devices concurrently), CUDA events on each launching
    stream; -> (max ms over devices and ranks, per-device ms)."""
    import torch

    for lg in legs:
        with torch.cuda.device(lg.dev):
            for _ in range(warmup):
                lg.launch()
    for lg in legs:
        torch.cuda.synchronize(lg.dev)
        lg.d_ev.zero_()
        torch.cuda.synchronize(lg.dev)
    devs.barrier()
    if clock is not None:
        clock.begin()
    for lg in legs:
        lg.e0.record(lg.stream)
    for _ in range(steps):
        for lg in legs:
            with torch.cuda.device(lg.dev):
                lg.launch()
    for lg in legs:
        lg.e1.record(lg.stream)
    for lg in legs:
        lg.stream.synchronize()
    if clock is not None:
        clock.end()
    devs.barrier()
    per = [lg.e0.elapsed_time(lg.e1) for lg in legs]
    return devs.max(max(per)), per


def pinned_empty(shape, dtype):
    import torch

    return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()


class HostBuffer:
    """An exact-size pinned host allocation from the library (sf_host_alloc: cudaHostAlloc), viewed
    as a numpy array -- torch's caching host allocator rounds up to a power of two, which at C5's
    90 GB would pin 128 GB."""

    def __init__(self, sf, shape, dtype):
        import ctypes

        self.L = sf._lib.lib()
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        self.ptr = self.L.sf_host_alloc(nbytes)
        if not self.ptr:
            raise MemoryError(f"sf_host_alloc({nbytes}) failed")
        buf = (ctypes.c_char * nbytes).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype).reshape(shape)

    def free(self):
        if self.ptr:
            self.array = None
            self.L.sf_host_free(self.ptr)
            self.ptr = None


def pinned_result(sf, count, P):
    import torch

    return sf.BatchResult(pinned_empty((count, P), torch.float32), pinned_empty(count, torch.float32),
                          pinned_empty(count, torch.float32), pinned_empty(count, torch.float32),
                          pinned_empty(count, torch.uint8), pinned_empty(count, torch.uint8))


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    import paper_2106_02045_b200 as sf

    devs = Devices(args)
    rank = devs.rank
    W, H, count, model = CONFIGS[args.config]
    count = args.count or count
    N = W * H
    result = {}

    # ---- headline: kernel-only fits/s on HBM-resident spots, every device at once (weak scaling)
    t0 = time.perf_counter()
    batches = []  # (device, images (host), d_img, d_ini)
    for k, d in enumerate(devs.ids):
        first = (rank * len(devs.ids) + k) * count  # global spot index of this device's shard
        batches.append((d,) + device_batch(sf, d, W, H, count, model, first))
    setup_s = time.perf_counter() - t0
    legs = [KernelLeg(sf, d, W, H, count, model, d_img, d_ini) for d, _, d_img, d_ini in batches]
    clock = ClockSampler(devs.ids)
    with clock:  # started (and live) before the warm-up; the summary keeps the timed window's rows
        ms_max, per_dev = time_legs(legs, args.steps, args.warmup, devs, clock)
    value = devs.n_gpus * count * args.steps / (ms_max * 1e-3)
    evs = [v / max(1, args.steps) for v in legs[0].d_ev.cpu().tolist()]  # per launch (= per step), device 0
    if args.profile:  # ncu / quick-look runs: kernel leg only (numbers taken under a profiler are not bench values)
        if rank == 0:
            print(json.dumps({"profile_only": True, "ms_per_step": ms_max / args.steps, "fits_per_s": value,
                              "evals": evs, "count": count, "per_device_ms": per_dev}))
        devs.close()
        return 0

    # ---- parity of the headline run (rank 0, device 0): sample vs the C oracle
    if rank == 0:
        _, images0, _, d_ini0 = batches[0]
        idx = np.linspace(0, count - 1, min(count, args.parity_sample)).astype(np.int64)
        result["parity"] = parity(legs[0].results(idx), images0[idx], d_ini0.cpu().numpy()[idx], W, H)
        result["initializer"] = initializer_leg(sf, devs.ids[0], batches[0][2], W, H, count, model)
    del legs

    # ---- end to end through the public API from host memory (all devices of this process)
    result.update(e2e_legs(sf, args, devs, batches, W, H, count, model))
    ini0 = batches[0][3].cpu().numpy()
    images0 = batches[0][1]
    del batches
    torch.cuda.empty_cache()

    # ---- BASELINE configs 1, 3, 4 (+ explicit-5) on device 0 of rank 0: kernel fits/s, roofline, parity
    if rank == 0 and args.per_config and args.config == "c2":
        result["per_config"] = per_config(sf, args, devs.ids[0])
        torch.cuda.empty_cache()
    devs.barrier()

    # ---- C5: 1e8 spots in total from pinned host memory, sharded over every GPU of the job
    if args.c5_spots > 0 and args.config == "c2":
        result["c5"] = c5_leg(sf, args, devs)
        torch.cuda.empty_cache()
    if rank == 0 and args.rt_frames > 0:
        result.setdefault("c5", {})["realtime"] = realtime(args, devs.ids[0], zero_copy=not args.rt_copy)

    # ---- CPU baselines (rank 0): the reference CPU fitter and the bit-exact C port on a bounded sample
    if rank == 0:
        cores = len(os.sched_getaffinity(0))
        samp = args.ref_sample or max(4000, 1500 * cores)
        cpu_v, cpu_dt, kind = cpu_reference(W, H, model, images0, ini0, samp, cores)
        c_v = cpu_c_port(W, H, images0, ini0, min(count, 20 * samp), cores)
        src = ("the unmodified reference spotfit.model (baseline/_ref)" if kind == "reference"
               else "oracle/model_np.py (restated reference numpy arithmetic)")
        result["cpu_baseline"] = {"value": cpu_v, "unit": "fits/s", "cores": cores, "kind": kind, "host": host_info(),
                                  "sample": f"spots 0..{samp - 1} of this workload, LM loop oracle/lm.py over {src}, "
                                            f"{cpu_dt:.1f} s wall on {cores} processes (~{cpu_dt * cores:.0f} s of "
                                            "CPU work)"}
        result["cpu_c_port"] = {"value": c_v, "unit": "fits/s", "cores": cores,
                                "note": "bit-exact C restatement (oracle/spotfit_oracle.c), stronger CPU comparator"}

    # ---- roofline of the headline kernel (device 0): algorithmic FP32 ops per launch / kernel time
    launch_s = per_dev[0] * 1e-3 / args.steps
    peaks = load_peaks()
    clks = clock.summary()
    sm_max = clks.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(devs.ids[0]).multi_processor_count
    rf = roofline_of(model, N, count, evs, launch_s, sms, sm_max)
    n_g, n_t, n_k = evs
    exps = N * (n_g + n_t)
    sfu_peak = sms * 16 * sm_max * 1e6
    hbm_bytes = count * (4 * N + 4 * model) + count * (4 * model + 12 + 2)
    xu_per_pix = {3: 6 + 6 + 1, 4: 6 + 10 + 1, 5: 21 + 1}[model]
    xu_ops = N * n_k * xu_per_pix
    inst_per_fit = traffic = None
    try:  # warp instructions and DRAM bytes per fit from the committed ncu capture of this kernel (profiles/)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        if model == 3 and (W, H) == (15, 15):
            traffic = t["bytes_per_spot"] * count
            inst_per_fit = t.get("inst_per_spot")
    except (OSError, KeyError, ValueError):
        pass
    roofline = {"bound": "fp32", "achieved": rf["achieved"], "peak": rf["peak"], "unit": "TOP/s", "frac": rf["frac"],
                "traffic": traffic,
                "traffic_note": "DRAM bytes per launch (ncu dram__bytes_read+write, profiles/ncu_traffic.json) "
                                f"vs {hbm_bytes:.4g} algorithmic bytes",
                "ops_per_fit": rf["ops_per_fit"],
                "def": "SURVEY 8d: N*(67*n_G + 18*n_T) algorithmic ops per fit; peak = SMs*128*sm_max_mhz (FP32 lanes)",
                "sfu": {"achieved": exps / launch_s / 1e12, "peak": sfu_peak / 1e12, "frac": exps / launch_s / sfu_peak},
                "hbm": {"achieved": hbm_bytes / launch_s / 1e9, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                        "frac": (hbm_bytes / launch_s / 1e9) / peaks["hbm_gbs"] if peaks.get("hbm_gbs") else None,
                        "peak_source": "MEASURED_PEAKS.json (measured)"},
                "issue": None if inst_per_fit is None else {
                    "achieved": inst_per_fit * count / launch_s / 1e12, "peak": sms * 4 * sm_max * 1e6 / 1e12,
                    "unit": "Twarp-inst/s", "frac": inst_per_fit * count / launch_s / (sms * 4 * sm_max * 1e6),
                    "def": "warp instructions issued (ncu smsp__inst_executed per fit, profiles/ncu_traffic.json) "
                           "vs 1 per clock per SM sub-partition"},
                "xu": {"achieved": xu_ops / launch_s / 1e12, "peak": sms * 16 * sm_max * 1e6 / 1e12,
                       "frac": (xu_ops / launch_s) / (sms * 16 * sm_max * 1e6),
                       "def": "XU pipe (16/clk/SM, measured): F2F.F64.F32 widenings of the signed f64 addends + "
                              "MUFU.RCP, per pixel per fused evaluation"}}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "fits/s", "n_gpus": devs.n_gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (per-pixel) / f64 (sums)",
            "data": "synthetic (simulator SPEC.md:316-368, 400:40 counts, seeded), inits from the untimed GPU "
                    "initializer",
            "config": workload_config(args, devs.n_gpus),
            "per_device_ms_per_step": [m / args.steps for m in per_dev],
            "driver": "torchrun, one rank per GPU (gloo barrier / max only)" if devs.world > 1 else
                      f"one process, devices {devs.ids} (per-device streams, concurrent launches)",
            "roofline": roofline,
            "gpu_launches": args.steps * len(devs.ids) * devs.world,
            "evals_per_fit": rf["evals_per_fit"],
            "clocks": clks,
            "setup_s": setup_s,
        }
        line.update(result)
        print(json.dumps(line))
    devs.close()
    return 0


def e2e_legs(sf, args, devs, batches, W, H, count, model):
    """The public call fit_batch from host memory over this process's devices (one call spanning
    them: sf_fit_batch's one-thread-per-device shards), timed on the host clock around the blocking
    call, max over ranks.  Headline `e2e`: pinned images, inits=None (the fit kernel's fused
    initializer), pinned outputs.  Variants: with inits (the paper's H2D + kernel + D2H span),
    pageable numpy (the plain drop-in caller), uint16 counts."""
    import torch

    nd = len(devs.ids)
    images = np.concatenate([b[1] for b in batches]) if nd > 1 else batches[0][1]
    inits = np.concatenate([b[3].cpu().numpy() for b in batches])
    total = images.shape[0]
    pin_img = torch.from_numpy(images).pin_memory().numpy()
    pin_ini = torch.from_numpy(inits).pin_memory().numpy()
    outs = pinned_result(sf, total, model)
    steps = max(3, args.steps // 2)
    npx = W * H
    d2h = total * (model * 4 + 3 * 4 + 2)
    call = dict(config=sf.FitConfig(), engine=ENGINE[model], grid=sf.PixelGrid(W, H), devices=devs.ids)

    def timed(fn):
        fn()  # warm-up (staging buffers, streams)
        s = 0.0
        r = None
        for _ in range(steps):
            devs.barrier()
            a = time.perf_counter()
            r = fn()
            s += devs.max(time.perf_counter() - a)
        return devs.n_gpus * count * steps / s, r

    def h2d(r):  # bytes the library actually copied host -> device in one call (sf_stats.h2d_bytes)
        return int(r.stats.get("h2d_bytes") or 0)

    v_fused, r = timed(lambda: sf.fit_batch(pin_img, None, out=outs, **call))
    res = {"e2e": {"value": v_fused, "unit": "fits/s", "h2d_bytes_per_step": h2d(r), "d2h_bytes_per_step": d2h,
                   "input_bytes_per_step": total * npx * 4, "steps": steps,
                   "chunks_per_step": r.stats.get("n_chunks"), "chunks_u16_per_step": r.stats.get("n_chunks_u16"),
                   "path": "fit_batch(pinned f32 images) -> sf_fit_batch, inits=None: integer-valued chunks narrowed "
                           "losslessly to u16 by the host (half the PCIe bytes; h2d_bytes_per_step counts what "
                           "crossed), initializer on the device, chunked H2D/kernel/D2H on "
                           f"{nd} device(s) of this process"}}
    keep = min(total, 50_000)
    fused = {k: np.array(getattr(outs, k)[:keep]) for k in FIELDS}
    v_in, r_in = timed(lambda: sf.fit_batch(pin_img, pin_ini, out=outs, **call))
    same = all(np.array_equal(fused[k].view(np.uint8), np.asarray(getattr(outs, k)[:keep]).view(np.uint8))
               for k in FIELDS)
    variants = {"pinned_with_inits": {"value": v_in, "unit": "fits/s",
                                      "h2d_bytes_per_step": h2d(r_in), "d2h_bytes_per_step": d2h,
                                      "path": "fit_batch(pinned images, pinned inits, out=pinned): the paper's span "
                                              "(PAPER.md:210, init excluded)"},
                "fused_equals_explicit_inits": {"spots": keep, "bitwise": bool(same)}}
    v_pg, r_pg = timed(lambda: sf.fit_batch(images, None, **call))
    variants["pageable_no_inits"] = {"value": v_pg, "unit": "fits/s", "h2d_bytes_per_step": h2d(r_pg),
                                     "d2h_bytes_per_step": d2h,
                                     "path": "fit_batch(numpy images): pageable in, new result arrays out, fused "
                                             "initializer (the plain drop-in call)"}
    if np.array_equal(images, np.round(images)) and images.max(initial=0) < 65536 and images.min(initial=0) >= 0:
        pin_u16 = torch.from_numpy(images.astype(np.uint16)).pin_memory().numpy()
        v16, _ = timed(lambda: sf.fit_batch(pin_u16, None, out=outs, **call))
        variants["u16_pinned_no_inits"] = {
            "value": v16, "unit": "fits/s", "h2d_bytes_per_step": total * npx * 2, "d2h_bytes_per_step": d2h,
            "path": "fit_batch(pinned uint16 counts) -> sf_fit_batch_u16 (half the PCIe bytes; staged as u16 and "
                    "widened in the fit kernel), fused initializer"}
    # the same call on pixels that do not narrow (every value + 0.5): f32 crosses PCIe, after the first
    # chunk's narrowing pass gives up at its first value
    frac_img = pin_img  # reuse the pinned buffer: +0.5 in place, restored below
    frac_img += np.float32(0.5)
    v_fr, r_fr = timed(lambda: sf.fit_batch(frac_img, None, out=outs, **call))
    frac_img -= np.float32(0.5)
    variants["pinned_fractional_no_inits"] = {
        "value": v_fr, "unit": "fits/s", "h2d_bytes_per_step": h2d(r_fr), "d2h_bytes_per_step": d2h,
        "chunks_u16_per_step": r_fr.stats.get("n_chunks_u16"),
        "path": "fit_batch(pinned f32 images + 0.5): nothing narrows, f32 over PCIe (speed only, no parity)"}
    res["e2e_variants"] = variants
    return res


def per_config(sf, args, dev):
    """BASELINE configs 1, 3, 4 and the explicit-5 baseline on one device: kernel-only fits/s
    (HBM-resident, device simulator + standalone initializer, untimed), FP32 roofline fraction and
    a bitwise parity sample against the C oracle."""
    import torch

    out = {}
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_max = load_peaks().get("sm_max_mhz") or 1965.0
    for name in [c for c in args.per_config.split(",") if c]:
        W, H, count, model = CONFIGS[name]
        if name == "c4" and args.c4_spots:
            count = args.c4_spots
        t0 = time.perf_counter()
        _, d_img, d_ini = device_batch(sf, dev, W, H, count, model, 0, host=False)
        setup = time.perf_counter() - t0
        leg = KernelLeg(sf, dev, W, H, count, model, d_img, d_ini)
        steps = 20 if count <= 100_000 else 3
        ms, _ = time_legs([leg], steps, 2, _Single())
        evs = [v / steps for v in leg.d_ev.cpu().tolist()]
        rf = roofline_of(model, W * H, count, evs, ms * 1e-3 / steps, sms, sm_max)
        # parity: first, last and evenly spaced spots vs the C oracle
        idx = np.unique(np.concatenate([np.linspace(0, count - 1, min(count, max(2, args.parity_sample // 4))),
                                        [0, count - 1]]).astype(np.int64))
        ti = torch.from_numpy(idx).to(dev)
        images = d_img.index_select(0, ti).cpu().numpy()
        inits = d_ini.index_select(0, ti).cpu().numpy()
        par = parity(leg.results(idx), images, inits, W, H)
        ini_leg = initializer_leg(sf, dev, d_img, W, H, count, model, reps=5 if count > 1_000_000 else 10)
        out[name] = {"workload": f"{count} {MODEL_NAME[model]} spots, {W}x{H} px", "spots": count,
                     "value": count * steps / (ms * 1e-3), "unit": "fits/s", "ms_per_step": ms / steps,
                     "steps": steps, "roofline_frac": rf["frac"], "ops_per_fit": rf["ops_per_fit"],
                     "evals_per_fit": rf["evals_per_fit"], "parity": par, "setup_s": setup,
                     "input_bytes": count * W * H * 4,
                     "initializer": {k: ini_leg[k] for k in ("ms_per_launch", "achieved_GBps", "frac")}}
        del leg, d_img, d_ini
        torch.cuda.empty_cache()
    return out


def c5_leg(sf, args, devs):
    """BASELINE configs[4]: 1e8 15x15 spots in total (strong scaling: each rank takes 1/world of
    them and drives its device(s); one process spans its devices through sf_fit_batch's shards),
    streamed from pinned host memory through the public call fit_batch(images) -- fused initializer,
    H2D + kernel + D2H -- with a bitwise parity sample around every shard boundary."""
    import torch

    W = H = 15
    N = W * H
    total = args.c5_spots
    lo = total * devs.rank // devs.world
    n = total * (devs.rank + 1) // devs.world - lo
    per_spot = N * 4 + 26
    avail = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_AVPHYS_PAGES") / max(1, devs.world)
    note = None
    if n * per_spot * 1.1 > 0.75 * avail:  # host memory cap: shrink (and say so) rather than swap / OOM the box
        n2 = max(1_000_000, int(0.75 * avail / (per_spot * 1.1)) // 1_000_000 * 1_000_000)
        note = f"host memory: {avail / 1e9:.0f} GB available to this rank, ran {n2} of its {n} spots"
        n = n2
    t0 = time.perf_counter()
    hb = HostBuffer(sf, (n, N), np.float32)
    images = hb.array
    outs = pinned_result(sf, n, 3)
    alloc_s = time.perf_counter() - t0
    # fill from the device generator in 1e6-spot pieces (global indices lo..lo+n-1, seed SEED)
    dev0 = devs.ids[0]
    piece = 1_000_000
    t0 = time.perf_counter()
    with torch.cuda.device(dev0):
        for a in range(0, n, piece):
            b = min(n, a + piece)
            d, _ = sf.simulate_batch_device(sf.SimConfig(width=W, height=H, count=b - a, seed=SEED),
                                            first_index=lo + a, device=dev0)
            torch.from_numpy(images[a:b]).copy_(d.reshape(b - a, N))
        torch.cuda.synchronize(dev0)
    gen_s = time.perf_counter() - t0
    grid = sf.PixelGrid(W, H)
    sf.fit_batch(images[: min(n, 200_000)], None, grid=grid, devices=devs.ids)  # warm-up (contexts, staging)
    steps = max(1, args.c5_steps)
    s = 0.0
    r = None
    for _ in range(steps):
        devs.barrier()
        a = time.perf_counter()
        r = sf.fit_batch(images, None, grid=grid, devices=devs.ids, out=outs)
        s += devs.max(time.perf_counter() - a)
    fits = devs.sum(float(n))
    res = {"spots": int(fits), "n_gpus": devs.n_gpus, "value": fits * steps / s, "unit": "fits/s", "steps": steps,
           "s_per_step": s / steps, "scaling": "strong (fixed total of spots)",
           "h2d_bytes_per_step": int(devs.sum(float(r.stats.get("h2d_bytes") or 0))),
           "input_bytes_per_step": int(fits) * N * 4, "d2h_bytes_per_step": int(fits) * 26,
           "path": "fit_batch(pinned numpy images, inits=None, out=pinned) -> sf_fit_batch(devices=all of this "
                   "process): contiguous shards, one host thread per device, integer-valued chunks narrowed to "
                   "u16 by the host, chunked H2D/kernel/D2H, initializer on the device",
           "chunks_per_step": r.stats.get("n_chunks"), "pinned_alloc_s": alloc_s, "generate_s": gen_s,
           "data": f"device simulator, seed {SEED}, global spot indices {lo}..{lo + n - 1} on rank {devs.rank}"}
    if note:
        res["note"] = note
    if devs.rank == 0:
        from oracle import initializer as oinit

        nd = len(devs.ids)
        bounds = [n * k // nd for k in range(1, nd)]  # sf_fit_batch's shard boundaries in this process
        near = (np.concatenate([np.arange(max(0, b - 3), min(n, b + 3)) for b in bounds]) if bounds
                else np.zeros(0, np.int64))
        idx = np.unique(np.concatenate([np.linspace(0, n - 1, max(2, args.parity_sample // 10)), near, [0, n - 1]])
                        .astype(np.int64))
        sample = images[idx]
        ini, _ = oinit.estimate_initial_batch_np(sample, W, H, 0.3, 15.0, 3)
        res["parity"] = parity({k: np.asarray(getattr(outs, k))[idx] for k in FIELDS}, sample, ini, W, H)
        res["parity"]["shard_boundaries"] = bounds
        res["parity"]["inits"] = "oracle/initializer.py on the sample (the product used its fused initializer)"
    del images, outs
    hb.free()
    return res


def realtime(args, dev, zero_copy=True):
    """C5 real-time mode (BASELINE.json configs[4]): 50 spots/frame, 1000 frames,
    per-frame latency of host frame -> LM fit -> results on the host,
    replayed as one CUDA graph per frame (host clock around each blocking frame).
    The fit kernel estimates the inits itself (fused initializer).  zero_copy: it
    reads the frame from, and writes the results to, pinned (device-mapped) host
    memory, so the graph is one kernel node; otherwise an explicit H2D copy, the
    kernel on device buffers and D2H copies."""
    import ctypes

    import torch

    import paper_2106_02045_b200 as sf
    from paper_2106_02045_b200 import _lib

    W = H = 15
    spf, frames = args.rt_spots, args.rt_frames
    grid = sf.PixelGrid(W, H)
    ccfg = sf.FitConfig().to_c(grid, 3)
    L = _lib.lib()
    allimg, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=spf * frames, seed=4242))
    allimg = allimg.reshape(frames, spf, W * H)
    with torch.cuda.device(dev):
        pin_in = torch.empty((spf, W * H), dtype=torch.float32).pin_memory()
        pin_u8 = torch.empty((2, spf), dtype=torch.uint8).pin_memory()
        d_img = torch.empty((spf, W * H), dtype=torch.float32, device=dev)
        d_par = torch.empty((spf, 3), dtype=torch.float32, device=dev)
        d_u8 = torch.empty((2, spf), dtype=torch.uint8, device=dev)
        d_ab = torch.empty((3, spf), dtype=torch.float32, device=dev)
        stream = torch.cuda.Stream(dev)
        h_ab = torch.empty((3, spf), dtype=torch.float32).pin_memory()
        h_par = torch.empty((spf, 3), dtype=torch.float32).pin_memory()

        # inits NULL: the fit kernel estimates each spot's init from the pixels it stages (fused initializer)
        def frame_ops_zero_copy():
            st = torch.cuda.current_stream(dev).cuda_stream
            _lib.check(L.sf_fit_batch_device(pin_in.data_ptr(), W, H, spf, None, ctypes.byref(ccfg),
                                             h_par.data_ptr(), h_ab[0].data_ptr(), h_ab[1].data_ptr(),
                                             h_ab[2].data_ptr(), pin_u8[0].data_ptr(), pin_u8[1].data_ptr(), None, st))

        def frame_ops_copy():
            st = torch.cuda.current_stream(dev).cuda_stream
            d_img.copy_(pin_in, non_blocking=True)
            _lib.check(L.sf_fit_batch_device(d_img.data_ptr(), W, H, spf, None, ctypes.byref(ccfg),
                                             d_par.data_ptr(), d_ab[0].data_ptr(), d_ab[1].data_ptr(),
                                             d_ab[2].data_ptr(), d_u8[0].data_ptr(), d_u8[1].data_ptr(), None, st))
            h_par.copy_(d_par, non_blocking=True)
            h_ab.copy_(d_ab, non_blocking=True)
            pin_u8.copy_(d_u8, non_blocking=True)

        frame_ops = frame_ops_zero_copy if zero_copy else frame_ops_copy
        with torch.cuda.stream(stream):
            for _ in range(3):
                frame_ops()
        stream.synchronize()
        graph = None
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
                frame_ops()
            graph = g
        except Exception as e:  # keep measuring without a graph rather than failing the bench
            sys.stderr.write(f"realtime: graph capture failed ({e}); plain launches\n")
        lat = []
        for f in range(frames):
            t0 = time.perf_counter()
            pin_in.numpy()[:] = allimg[f]  # the camera frame lands in pinned staging
            with torch.cuda.stream(stream):  # CUDAGraph.replay launches on the current stream
                if graph is not None:
                    graph.replay()
                else:
                    frame_ops()
            stream.synchronize()
            lat.append(time.perf_counter() - t0)
        lat_us = np.array(lat) * 1e6
        # the last frame's results equal the batch API's on the same spots (bitwise)
        par, ab, u8 = h_par.numpy().copy(), h_ab.numpy().T.copy(), pin_u8.numpy().copy()
    ref = sf.fit_batch(allimg[frames - 1], grid=grid, devices=[dev])
    same = (np.array_equal(par.view(np.uint32), np.asarray(ref.params).view(np.uint32))
            and np.array_equal(ab[:, 0].view(np.uint32), np.asarray(ref.alpha).view(np.uint32))
            and np.array_equal(u8[0], np.asarray(ref.status)) and np.array_equal(u8[1], np.asarray(ref.iterations)))
    return {"spots_per_frame": spf, "frames": frames, "grid": f"{W}x{H}", "cuda_graph": graph is not None,
            "zero_copy": zero_copy, "matches_fit_batch": bool(same),
            "p50_us": float(np.percentile(lat_us, 50)), "p99_us": float(np.percentile(lat_us, 99)),
            "max_us": float(lat_us.max()), "mean_us": float(lat_us.mean()),
            "sustains_1kHz": bool(np.percentile(lat_us, 99) < 1000.0),
            "span": ("host frame copy -> one fit kernel (fused initializer + LM) reading the pinned frame over PCIe "
                     "and writing the results to pinned host memory (blocking per frame)") if zero_copy else
                    "host frame copy -> H2D -> fit kernel (fused initializer + LM) -> D2H (blocking per frame)"}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1, help="GPUs this process drives (ignored under torchrun)")
    ap.add_argument("--devices", default="", help="explicit device ids, e.g. 0,0 to exercise two shards on one GPU")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--count", type=int, default=0, help="override spots per GPU")
    ap.add_argument("--ref-sample", type=int, default=0)
    ap.add_argument("--parity-sample", type=int, default=20000)
    ap.add_argument("--per-config", default="c1,c3,c4,c2x", help="'' disables the per-config legs")
    ap.add_argument("--c4-spots", type=int, default=0, help="override the c4 size (default 1e7)")
    ap.add_argument("--c5-spots", type=int, default=100_000_000, help="0 disables the C5 leg")
    ap.add_argument("--c5-steps", type=int, default=2)
    ap.add_argument("--profile", action="store_true", help="kernel leg only (for ncu); prints no bench line")
    ap.add_argument("--rt-spots", type=int, default=50, help="real-time mode: spots per frame (C5)")
    ap.add_argument("--rt-frames", type=int, default=1000, help="real-time mode frames (0 disables)")
    ap.add_argument("--rt-copy", action="store_true", help="real-time mode with explicit H2D/D2H copies")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
