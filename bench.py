"""bench.py -- headline benchmark: 2D Gaussian fits/s (15x15 px, symmetric,
implicit alpha/beta) on N B200s vs the reference CPU fitter.

Workload (BASELINE.json configs[1]): 1e6 synthetic spots per GPU,
15x15 px, 400:40 counts, Poisson-like noise, inits from the (untimed) GPU
initializer, exactly as PAPER.md:210-212 times the fit.  A step = one full LM
fit of the whole batch.

  value  -- fits/s with inputs resident in HBM (sf_fit_batch_device, CUDA
            events on the launching stream, max over ranks); 900 MB of input per
            GPU > 126 MB L2, so no L2 flush is needed between steps.
  e2e    -- the same fit through the public API (fit_batch -> sf_fit_batch)
            from pinned host memory: H2D + kernel + D2H inside the timed region.
  --impl reference -- the reference CPU fitter (numpy model arithmetic of
            pkg/src/spotfit/model.py restated in oracle/model_np.py + the App. A
            LM loop) on all host cores, bounded sample per step.

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
    "c4": (32, 32, 1_000_000, 3),
    "c2x": (15, 15, 1_000_000, 5),  # explicit 5-parameter baseline on the C2 workload
}
METRIC = "2D Gaussian fits/sec (15x15 px) at 1/2/4/8 B200 vs CPU ref; % FP32/SFU roofline"
# algorithmic work per pixel-evaluation: G-eval 67 ops (45 FP32 + 22 reduction adds),
# T-eval 18 ops (14 + 4); one exp each.  Elliptical G-eval: 58 + 30.
OPS_G = {3: 67, 4: 88, 5: 60}  # explicit-5: 39 FP32 + 21 reduction adds per pixel-evaluation (G = T)
OPS_T = {3: 18, 4: 18, 5: 60}


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
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def make_workload(W, H, count, model, seed):
    import paper_2106_02045_b200 as sf

    sim_model = 4 if model == 4 else 3  # explicit-5 fits symmetric spots
    im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=count, seed=seed, model=sim_model))
    return im.reshape(count, W * H)


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


def run_reference(args):
    rank, world, _ = dist_env()
    W, H, count, model = CONFIGS[args.config]
    if rank != 0:
        return 0
    import paper_2106_02045_b200 as sf  # simulator + (host) initializer inputs only
    from oracle import initializer as oinit

    cores = len(os.sched_getaffinity(0))
    sample = args.ref_sample or max(4000, 1500 * cores)
    images = make_workload(W, H, sample, model, seed=2021)
    inits, amps = oinit.estimate_initial_batch(images, W, H, 0.3, float(max(W, H)), min(model, 4))
    if model == 5:
        inits = np.concatenate([inits, amps], axis=1).astype(np.float32)
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
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic (SPEC.md:316-368 simulator, 400:40 counts)",
        "config": {"workload": f"{args.config}: {W}x{H} {'symmetric' if model == 3 else 'elliptical'}, "
                               f"bounded sample of {sample} spots per step", "spots_per_step": sample,
                   "cores": cores},
        "cpu_baseline": {"value": value, "unit": "fits/s", "cores": cores, "kind": kind, "host": host_info(),
                         "sample": f"{sample} spots of the {W}x{H} workload per step, {args.steps} steps; "
                                   "arithmetic: reference spotfit.model from baseline/_ref, LM loop oracle/lm.py"},
        "e2e": {"value": value, "unit": "fits/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def realtime(args, dev, zero_copy=True):
    """C5 real-time mode (BASELINE.json configs[4]): 50 spots/frame, 1000 frames,
    per-frame latency of host frame -> GPU initializer -> LM fit -> results on the host,
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
    cfg = sf.FitConfig()
    ccfg = cfg.to_c(grid, 3)
    b = cfg.resolved_bounds(grid)
    L = _lib.lib()
    allimg = make_workload(W, H, spf * frames, 3, seed=4242).reshape(frames, spf, W * H)
    pin_in = torch.empty((spf, W * H), dtype=torch.float32).pin_memory()
    pin_u8 = torch.empty((2, spf), dtype=torch.uint8).pin_memory()
    d_img = torch.empty((spf, W * H), dtype=torch.float32, device=dev)
    d_ini = torch.empty((spf, 3), dtype=torch.float32, device=dev)
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

    def frame_result():
        return h_par.numpy().copy(), h_ab.numpy().T.copy(), pin_u8.numpy().copy()

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
    par, ab, u8 = frame_result()
    ref = sf.fit_batch(allimg[frames - 1], grid=grid)
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


def run_ours(args):
    import torch

    import paper_2106_02045_b200 as sf
    from paper_2106_02045_b200 import _lib

    rank, world, local = dist_env()
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    dev = torch.cuda.current_device()
    if world > 1:
        import torch.distributed as dist

        # plumbing only (barrier + max-over-ranks timing): NCCL with one rank per GPU; gloo when ranks share a
        # GPU (SPOTFIT_DIST_BACKEND=gloo, used to exercise this path on a single-GPU box)
        backend = os.environ.get("SPOTFIT_DIST_BACKEND", "nccl" if ndev >= world else "gloo")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev if torch.distributed.get_backend() == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())
    W, H, count, model = CONFIGS[args.config]
    if args.count:
        count = args.count
    N = W * H
    grid = sf.PixelGrid(W, H)
    cfg = sf.FitConfig()
    ccfg = cfg.to_c(grid, model)
    L = _lib.lib()

    # ---- synthetic inputs (untimed): simulator -> HBM; GPU initializer (untimed)
    t0 = time.perf_counter()
    images = make_workload(W, H, count, model, seed=1000 + rank)
    d_img = torch.from_numpy(images).to(dev)
    d_ini = sf.batch_engine._auto_inits(d_img, grid, model, cfg)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    d_par = torch.empty((count, model), dtype=torch.float32, device=dev)
    d_f = torch.empty((3, count), dtype=torch.float32, device=dev)
    d_u8 = torch.empty((2, count), dtype=torch.uint8, device=dev)
    d_ev = torch.zeros(3, dtype=torch.int64, device=dev)
    stream = torch.cuda.Stream(dev)

    def step():
        rc = L.sf_fit_batch_device(d_img.data_ptr(), W, H, count, d_ini.data_ptr(), ctypes_byref(ccfg),
                                   d_par.data_ptr(), d_f[0].data_ptr(), d_f[1].data_ptr(), d_f[2].data_ptr(),
                                   d_u8[0].data_ptr(), d_u8[1].data_ptr(), d_ev.data_ptr(), stream.cuda_stream)
        _lib.check(rc)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    stream.synchronize()
    d_ev.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        stream.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    evs = d_ev.cpu().tolist()
    ms_max = max_over_ranks(ms)
    fits = count * world * args.steps
    value = fits / (ms_max * 1e-3)

    if args.profile:  # ncu / quick-look runs: kernel leg only (numbers taken under a profiler are not bench values)
        if rank == 0:
            print(json.dumps({"profile_only": True, "ms_per_step": ms_max / args.steps, "fits_per_s": value,
                              "evals": evs, "count": count}))
        return 0

    # ---- end to end through the public API from pinned host memory
    pin_img = torch.from_numpy(images).pin_memory()
    pin_ini = d_ini.cpu().pin_memory()
    outs = sf.BatchResult(*[torch.empty(s, dtype=d).pin_memory().numpy() for s, d in [
        ((count, model), torch.float32), (count, torch.float32), (count, torch.float32), (count, torch.float32),
        (count, torch.uint8), (count, torch.uint8)]])
    engine = {3: "implicit3", 4: "elliptical", 5: "explicit5"}[model]
    for _ in range(max(1, args.warmup)):
        sf.fit_batch(pin_img.numpy(), pin_ini.numpy(), config=cfg, engine=engine, grid=grid, out=outs, devices=[dev])
    barrier()
    e2e_steps = max(3, args.steps // 2)
    chunks = 0
    e2e_s = 0.0
    for _ in range(e2e_steps):  # blocking public call: host clock, max over ranks per step
        barrier()
        a = time.perf_counter()
        r = sf.fit_batch(pin_img.numpy(), pin_ini.numpy(), config=cfg, engine=engine, grid=grid, out=outs,
                         devices=[dev])
        e2e_s += max_over_ranks(time.perf_counter() - a)
        chunks = r.stats["n_chunks"]
    e2e_value = count * world * e2e_steps / e2e_s
    # the same public call with 16-bit camera counts (sf_fit_batch_u16: half the PCIe bytes, staged as u16
    # and widened by the fit kernel); reported beside the headline, which streams the reference's float32 layout
    e2e_u16 = None
    if np.array_equal(images, np.round(images)) and images.max(initial=0) < 65536 and images.min(initial=0) >= 0:
        pin_u16 = torch.from_numpy(images.astype(np.uint16)).pin_memory()
        sf.fit_batch(pin_u16.numpy(), pin_ini.numpy(), config=cfg, engine=engine, grid=grid, out=outs, devices=[dev])
        u16_s = 0.0
        for _ in range(e2e_steps):
            barrier()
            a = time.perf_counter()
            sf.fit_batch(pin_u16.numpy(), pin_ini.numpy(), config=cfg, engine=engine, grid=grid, out=outs,
                         devices=[dev])
            u16_s += max_over_ranks(time.perf_counter() - a)
        e2e_u16 = {"value": count * world * e2e_steps / u16_s, "unit": "fits/s",
                   "h2d_bytes_per_step": count * (N * 2 + model * 4), "d2h_bytes_per_step": count * (model * 4 + 14),
                   "path": "fit_batch(uint16 images) -> sf_fit_batch_u16 (u16 over PCIe, staged as u16 and widened in the fit kernel)"}

    # ---- parity on a sample (GPU vs C oracle, bitwise) and CPU baselines (rank 0)
    result = {}
    if rank == 0 and args.rt_frames > 0:
        result["realtime"] = realtime(args, dev, zero_copy=not args.rt_copy)
    if rank == 0:
        from oracle import lm, oracle_c

        par = d_par.cpu().numpy()
        f = d_f.cpu().numpy()
        u8 = d_u8.cpu().numpy()
        ini = d_ini.cpu().numpy()
        sample_idx = np.linspace(0, count - 1, min(count, args.parity_sample)).astype(np.int64)
        ref = oracle_c.fit_batch(images[sample_idx], ini[sample_idx], W, H, lm.LMConfig.for_grid(W, H))
        same = np.ones(len(sample_idx), bool)
        for k, got in (("params", par[sample_idx]), ("alpha", f[0][sample_idx]), ("beta", f[1][sample_idx]),
                       ("nchi2", f[2][sample_idx]), ("status", u8[0][sample_idx]),
                       ("iterations", u8[1][sample_idx])):
            eq = (np.asarray(got).view(np.uint8).reshape(len(sample_idx), -1) ==
                  np.asarray(ref[k]).view(np.uint8).reshape(len(sample_idx), -1)).all(axis=1)
            same &= eq
        result["parity"] = {"sample": int(len(sample_idx)), "bitwise_identical_frac": float(same.mean()),
                            "state_identical_frac": float((u8[0][sample_idx] == ref["status"]).mean()),
                            "checker": "oracle/spotfit_oracle.c (pinned to reference model.py fixtures)"}
        cores = len(os.sched_getaffinity(0))
        samp = args.ref_sample or max(4000, 1500 * cores)
        cpu_v, cpu_dt, kind = cpu_reference(W, H, model, images, ini, samp, cores)
        c_v = cpu_c_port(W, H, images, ini, min(count, 20 * samp), cores)
        src = ("the unmodified reference spotfit.model (baseline/_ref)" if kind == "reference"
               else "oracle/model_np.py (restated reference numpy arithmetic)")
        result["cpu_baseline"] = {"value": cpu_v, "unit": "fits/s", "cores": cores, "kind": kind, "host": host_info(),
                                  "sample": f"{samp} spots of this workload, LM loop oracle/lm.py over {src}, "
                                            f"{cpu_dt:.1f} s wall on {cores} processes (~{cpu_dt * cores:.0f} s of CPU work)"}
        result["cpu_c_port"] = {"value": c_v, "unit": "fits/s", "cores": cores,
                                "note": "bit-exact C restatement (oracle/spotfit_oracle.c), stronger CPU comparator"}

    # ---- roofline: algorithmic FP32 ops per launch / kernel time
    n_g, n_t, n_k = (v / max(1, args.steps) for v in evs)  # per launch (= per step)
    ops = N * (OPS_G[model] * n_g + OPS_T[model] * n_t)
    exps = N * (n_g + n_t)
    launch_s = ms * 1e-3 / args.steps
    peaks = load_peaks()
    clks = clk.summary()
    sm_max = clks.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    fp32_peak = sms * 128 * sm_max * 1e6
    sfu_peak = sms * 16 * sm_max * 1e6
    achieved = ops / launch_s
    hbm_bytes = count * (4 * N + 4 * model) + count * (4 * model + 12 + 2)
    # XU-pipe ops per pixel per fused evaluation (tame spots): the F2F.F64.F32
    # widenings of the signed addends (non-negative ones take IMAD.WIDE) + 1 MUFU.RCP of the exp
    xu_per_pix = {3: 6 + 6 + 1, 4: 6 + 10 + 1, 5: 21 + 1}[model]
    xu_ops = N * n_k * xu_per_pix
    inst_per_fit = None  # warp instructions per fit from the committed ncu capture (profiles/ncu_traffic.json)
    traffic = None  # DRAM bytes per launch from the committed ncu capture of this kernel (profiles/)
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        if model == 3 and (W, H) == (15, 15):
            traffic = t["bytes_per_spot"] * count
            inst_per_fit = t.get("inst_per_spot")
    except (OSError, KeyError, ValueError):
        pass
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "fits/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (per-pixel) / f64 (sums)",
            "data": "synthetic (simulator SPEC.md:316-368, 400:40 counts, seeded), inits from the untimed GPU initializer",
            "config": {"workload": f"{args.config}: {count} {'symmetric' if model == 3 else 'elliptical'} spots/GPU, "
                                   f"{W}x{H} px, max 20 LM iterations", "spots_per_gpu": count, "W": W, "H": H,
                       "model": model, "parallelism": f"independent shards x{world}",
                       "l2": f"inputs {count * N * 4 / 1e6:.0f} MB/GPU > 126 MB L2 (no flush needed)"},
            "roofline": {"bound": "fp32", "achieved": achieved / 1e12, "peak": fp32_peak / 1e12, "unit": "TOP/s",
                         "frac": achieved / fp32_peak, "traffic": traffic,
                         "traffic_note": "DRAM bytes per launch (ncu dram__bytes_read+write, profiles/ncu_traffic.json) "
                                         f"vs {hbm_bytes:.4g} algorithmic bytes",
                         "ops_per_fit": ops / count, "def": "SURVEY 8d: N*(67*n_G + 18*n_T) algorithmic ops per fit; "
                                                            "peak = SMs*128*sm_max_mhz (FP32 lanes)",
                         "sfu": {"achieved": exps / launch_s / 1e12, "peak": sfu_peak / 1e12,
                                 "frac": exps / launch_s / sfu_peak},
                         "hbm": {"achieved": hbm_bytes / launch_s / 1e9, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                                 "frac": (hbm_bytes / launch_s / 1e9) / peaks["hbm_gbs"] if peaks.get("hbm_gbs") else None,
                                 "peak_source": "MEASURED_PEAKS.json (measured)"},
                         "issue": None if inst_per_fit is None else {
                             "achieved": inst_per_fit * count / launch_s / 1e12, "peak": sms * 4 * sm_max * 1e6 / 1e12,
                             "unit": "Twarp-inst/s",
                             "frac": inst_per_fit * count / launch_s / (sms * 4 * sm_max * 1e6),
                             "def": "binding resource: warp instructions issued (ncu smsp__inst_executed per fit, "
                                    "profiles/ncu_traffic.json) vs 1 per clock per SM sub-partition"},
                         "xu": {"achieved": xu_ops / launch_s / 1e12, "peak": sms * 16 * sm_max * 1e6 / 1e12,
                                "frac": (xu_ops / launch_s) / (sms * 16 * sm_max * 1e6),
                                "def": "XU pipe (16/clk/SM, measured): F2F.F64.F32 widenings of the signed f64 "
                                       "addends + MUFU.RCP, per pixel per fused evaluation"}},
            "e2e": {"value": e2e_value, "unit": "fits/s", "h2d_bytes_per_step": count * (N + model) * 4,
                    "d2h_bytes_per_step": count * (model * 4 + 3 * 4 + 2), "steps": e2e_steps,
                    "path": "fit_batch -> sf_fit_batch, pinned host buffers, chunked H2D/kernel/D2H",
                    "chunks_per_step": chunks},
            "e2e_u16": e2e_u16,
            "gpu_launches": args.steps,
            "evals_per_fit": {"n_G": n_g / count, "n_T": n_t / count, "kernel": n_k / count},
            "clocks": clks,
            "setup_s": setup_s,
        }
        line.update(result)
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def ctypes_byref(x):
    import ctypes

    return ctypes.byref(x)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--count", type=int, default=0, help="override spots per GPU")
    ap.add_argument("--ref-sample", type=int, default=0)
    ap.add_argument("--parity-sample", type=int, default=20000)
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
