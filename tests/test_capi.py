"""C-ABI surface (CPU): the library loads, exports every symbol include/spotfit.h
declares, validates arguments, maps lanes onto numpy's pairwise tree, and
fails loudly (no CPU fallback) when no GPU is present."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def L():
    from paper_2106_02045_b200 import _lib

    return _lib.lib()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "spotfit.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(sf_[a-z_0-9]+)\s*\(", hdr)))


def test_exports_every_declared_symbol(L):
    from paper_2106_02045_b200 import _lib

    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.SYMBOLS), "ctypes table out of sync with include/spotfit.h"


def test_version_and_struct_layout(L):
    from paper_2106_02045_b200 import _lib
    from paper_2106_02045_b200.model import EVAL_DTYPE

    assert L.sf_version() == 1
    assert ctypes.sizeof(_lib.sf_eval_record) == EVAL_DTYPE.itemsize
    assert ctypes.sizeof(_lib.sf_config) == 8 + 11 * 8


def test_ctypes_structs_mirror_the_header():
    """Every C struct of include/spotfit.h and its ctypes mirror in _lib.py: same field names in the
    same order (the ABI the reference-side binding in INTEGRATION.md relies on)."""
    from paper_2106_02045_b200 import _lib

    hdr = open(os.path.join(ROOT, "include", "spotfit.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    for name in ("sf_stats", "sf_config"):
        body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), hdr, re.S).group(1)
        fields = []
        for decl in body.split(";"):
            decl = decl.strip()
            if decl:
                fields += [f.strip() for f in re.sub(r"^[\w\s]*?\b(?:u?int\d+_t|double|float|int)\b", "", decl).split(",")]
        assert [f for f, _ in getattr(_lib, name)._fields_] == fields, name


def test_lane_geometry_reproduces_numpy_pairwise_order(L):
    """Emulate the kernel's reduction (chain lanes -> xor 1,2,4 -> leaf tails ->
    slot butterfly -> 0.0 +) with the C++ lane geometry and compare with
    ndarray.sum(dtype=float64) for every N in 1..1024."""
    rng = np.random.default_rng(0)
    for N in range(1, 1025):
        slots = ctypes.c_int32()
        ppl = ctypes.c_int32()
        nc, nt, base, tbase = (np.zeros(128, np.int16) for _ in range(4))
        assert L.sf_lane_geometry(N, 1, ctypes.byref(slots), ctypes.byref(ppl), nc.ctypes.data, nt.ctypes.data,
                                  base.ctypes.data, tbase.ctypes.data) == 0
        S = slots.value
        assert S in (1, 2, 4, 8, 16) and 1 <= ppl.value <= 22
        x = (rng.standard_normal(N) * 10.0 ** rng.uniform(-5, 5, N)).astype(np.float32)
        lanes = 8 * S
        acc = []
        for l in range(lanes):
            a = 0.0
            for j in range(nc[l]):
                v = float(x[base[l] + 8 * j])
                a = v if j == 0 else a + v
            acc.append(a)
        o = 1
        while o < 8:  # leaf combine
            acc = [acc[l] + acc[l ^ o] for l in range(lanes)]
            o <<= 1
        for l in range(lanes):  # serial tails
            for t in range(nt[l]):
                acc[l] = acc[l] + float(x[tbase[l] + t])
        o = 8
        while o < lanes:  # slot tree
            acc = [acc[l] + acc[l ^ o] for l in range(lanes)]
            o <<= 1
        total = 0.0 + acc[0]
        assert all(v == acc[0] for v in acc), N
        assert total == x.sum(dtype=np.float64), N
        covered = sorted([base[l] + 8 * j for l in range(lanes) for j in range(nc[l])] +
                         [tbase[l] + t for l in range(0, lanes, 8) for t in range(nt[l])])
        assert covered == list(range(N)), N


def test_rejects_bad_grids_and_configs(L):
    from paper_2106_02045_b200 import _lib

    assert L.sf_lane_geometry(33, 32, None, None, None, None, None, None) != 0
    assert b"exceeds 1024" in L.sf_last_error()
    assert L.sf_lane_geometry(0, 5, None, None, None, None, None, None) != 0
    cfg = _lib.sf_config(3, 0, 0.0, 1e-6, 1e-4, 0.01, 10, 10, 1e4, 4, 4, 0.3, 9)
    rc = L.sf_fit_batch_device(None, 9, 9, 1, None, ctypes.byref(cfg), None, None, None, None, None, None, None, None)
    assert rc != 0 and b"max_iterations" in L.sf_last_error()


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) not in (None,) and False, reason="")
def test_fails_loudly_without_gpu():
    """The product path has no CPU fallback (raises when no device is visible)."""
    import paper_2106_02045_b200 as sf
    from paper_2106_02045_b200 import _lib

    if _lib.lib().sf_device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.SpotfitError, match="no CUDA device"):
        sf.fit_batch(np.zeros((2, 9, 9), np.float32), np.tile(np.float32([4, 4, 1.5]), (2, 1)))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2106_02045_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert '#include "spotfit_oracle' not in src and "libspotfit_oracle" not in src, f
