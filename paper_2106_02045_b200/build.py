"""Build the sm_100a shared library libspotfit_b200.so in-tree.

nvcc only (no torch JIT, no cache outside the repo): the library must travel
to the GPU box inside the repo snapshot.  Template instantiation units
(csrc/sf_inst.cu, one per (P, SLOTS)) compile in parallel.

    python -m paper_2106_02045_b200.build [--force] [--jobs N]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.environ.get("SPOTFIT_CSRC") or os.path.join(PKG, "csrc")  # alternate tree for A/B builds
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(PKG, "_build")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libspotfit_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: no FMA contraction anywhere (the parity contract);
# explicit __fmaf_rn in npexp stays fused.  Denormals kept (no -ftz).
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                     "-Xptxas", "-v", f"-I{INCLUDE}", f"-I{CSRC}"]
UNITS = [(p, s) for p in (3, 4, 5) for s in (1, 2, 4, 8, 16)]
HEADERS = ["sf_device.cuh", "sf_fit_kernel.cuh", "sf_fit2l.cuh", "sf_init_core.cuh", "sf_launch.h", "sf_geometry.h", "sf_sim_core.h"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, log):
    p = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
    if p.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return p.stderr


def build(force: bool = False, jobs: int = 0, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Build the library; `variant` + `defines` produce an A/B build under
    _lib/variants/<variant>/ (select it at run time with SPOTFIT_LIB)."""
    obj = os.path.join(OBJ, "variants", variant) if variant else OBJ
    lib = os.path.join(LIBDIR, "variants", variant, "libspotfit_b200.so") if variant else LIB
    os.makedirs(obj, exist_ok=True)
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "spotfit.h"), __file__]
    tasks = []
    for p, s in UNITS:
        src = os.path.join(CSRC, "sf_inst.cu")
        out = os.path.join(obj, f"sf_inst_P{p}_S{s}.o")
        cmd = [nvcc()] + NVCC_FLAGS + dflags + [f"-DSF_P={p}", f"-DSF_SLOTS={s}", "-c", src, "-o", out]
        tasks.append((out, [src] + hdrs, cmd))
    for name in ("sf_init.cu", "sf_capi.cu", "sf_sim.cu", "sf_model.cu"):
        src = os.path.join(CSRC, name)
        out = os.path.join(obj, name.replace(".cu", ".o"))
        tasks.append((out, [src] + hdrs, [nvcc()] + NVCC_FLAGS + dflags + ["-c", src, "-o", out]))
    src = os.path.join(CSRC, "sf_sim.cpp")
    out = os.path.join(obj, "sf_sim_host.o")
    tasks.append((out, [src, os.path.join(CSRC, "sf_sim_core.h"), os.path.join(INCLUDE, "spotfit.h"), __file__],
                  ["g++", "-O2", "-fPIC", "-std=c++17", "-ffp-contract=off", "-pthread", f"-I{INCLUDE}", "-c", src,
                   "-o", out]))
    src = os.path.join(CSRC, "sf_host_narrow.cpp")
    out = os.path.join(obj, "sf_host_narrow.o")
    tasks.append((out, [src, os.path.join(INCLUDE, "spotfit.h"), __file__],
                  ["g++", "-O3", "-fPIC", "-std=c++17", "-pthread", f"-I{INCLUDE}"] + dflags + ["-c", src, "-o", out]))
    src = os.path.join(CSRC, "sf_csv.cpp")
    out = os.path.join(obj, "sf_csv_host.o")
    tasks.append((out, [src, os.path.join(CSRC, "sf_pow5_tables.h"), os.path.join(INCLUDE, "spotfit.h"), __file__],
                  ["g++", "-O3", "-fPIC", "-std=c++17", "-pthread", f"-I{INCLUDE}", f"-I{CSRC}", "-c", src,
                   "-o", out]))
    todo = [t for t in tasks if force or _stale(t[0], t[1])]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
            futs = [ex.submit(_run, cmd, out + ".log") for out, _, cmd in todo]
            for f in futs:
                err = f.result()
                if verbose:
                    sys.stderr.write(err)
    objs = [t[0] for t in tasks]
    if force or todo or _stale(lib, objs):
        _run([nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs + ["-lpthread"],
             os.path.join(obj, "link.log"))
    return lib


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=0)
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--variant", default="")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args(argv)
    print(build(force=a.force, jobs=a.jobs, verbose=a.verbose, variant=a.variant, defines=a.defines))


if __name__ == "__main__":
    main()
