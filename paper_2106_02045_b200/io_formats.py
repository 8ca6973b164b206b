"""File formats of the reference CLI: SPB1 spot batches and
ParamsCSV / truth CSV.

SPB1: magic "SPB1", u16 version = 1, u16 width, u16 height, u32 count, then
count*width*height little-endian float32 pixels, images concatenated in index
order, each row-major.  The field list of SPEC.md:520 adds up to a 14-byte
header; the size invariant of SPEC.md:521 ("12 + 4*count*width*height") is
inconsistent with it -- the explicit field layout is followed, so the file
size is 14 + 4*count*width*height.

ParamsCSV: header ``index,x,y,sigma,alpha,beta,status,iterations,nchi2``, one
row per fit sorted by index, status as the StopReason name, floats rendered as
the shortest string that round-trips the float32 value.  Truth files use
``index,x,y,sigma,alpha,beta``.  (Elliptical fits add sigma_y after sigma.)
"""
from __future__ import annotations

import ctypes
import os
import struct

import numpy as np

MAGIC = b"SPB1"
VERSION = 1
HEADER = struct.Struct("<4sHHHI")  # 12 bytes
STOP_NAMES = ["MaxError", "MinDelta", "MinStep", "NotConverged", "MaxIterations"]


class MalformedSPB1(ValueError):
    """Malformed SPB1 file; `offset` is the byte offset of the problem."""

    def __init__(self, msg: str, offset: int):
        super().__init__(f"{msg} (at byte offset {offset})")
        self.offset = offset


def write_spb1(path: str, images: np.ndarray) -> None:
    """images: (count, H, W) float32-convertible."""
    a = np.ascontiguousarray(images, dtype="<f4")
    if a.ndim != 3:
        raise ValueError("images must be (count, H, W)")
    count, H, W = a.shape
    if W < 1 or H < 1 or W * H > 1024:
        raise ValueError(f"grid {W}x{H} outside 1..1024 pixels")
    with open(path, "wb") as f:
        f.write(HEADER.pack(MAGIC, VERSION, W, H, count))
        f.write(a.tobytes())


def read_spb1(path: str, mmap: bool = True):
    """-> (images (count, H, W) float32 view, width, height).  Zero-copy memory map by default."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        head = f.read(HEADER.size)
    if len(head) < HEADER.size:
        raise MalformedSPB1("truncated header", len(head))
    magic, version, W, H, count = HEADER.unpack(head)
    if magic != MAGIC:
        raise MalformedSPB1(f"bad magic {magic!r}", 0)
    if version != VERSION:
        raise MalformedSPB1(f"unsupported version {version}", 4)
    if W < 1 or H < 1 or W * H > 1024:
        raise MalformedSPB1(f"grid {W}x{H} outside 1..1024 pixels", 6)
    want = HEADER.size + 4 * count * W * H
    if size != want:
        raise MalformedSPB1(f"file size {size} != {want} for {count} images of {W}x{H}", min(size, want))
    if count == 0:
        return np.zeros((0, H, W), np.float32), W, H
    if mmap:
        a = np.memmap(path, dtype="<f4", mode="r", offset=HEADER.size, shape=(count, H, W))
    else:
        a = np.fromfile(path, dtype="<f4", offset=HEADER.size).reshape(count, H, W)
    return a, W, H


def fmt32(values) -> list:
    """Shortest decimal strings that round-trip float32 values exactly."""
    return [np.format_float_positional(np.float32(v), unique=True, trim="-") if np.isfinite(v)
            else ("nan" if np.isnan(v) else ("inf" if v > 0 else "-inf")) for v in np.asarray(values, np.float32)]


def status_name(status: int) -> str:
    return STOP_NAMES[int(status) & 7]


# ---------------------------------------------------------------- native writer / reader
# Rows are rendered and parsed by the library's host code (csrc/sf_csv.cpp: Ryu shortest digits,
# multi-threaded blocks); fmt32 above is the numpy statement of the same rendering, used by the tests.

def _col(kind, arr, stride=1):
    from . import _lib

    return _lib.sf_csv_col(kind, arr.ctypes.data, stride)


def _csv_write(path_or_file, header, cols, keep, rows, first_index, threads):
    from . import _lib

    if hasattr(path_or_file, "write"):  # file object: render into a temporary file, then copy the text
        import tempfile

        with tempfile.TemporaryDirectory() as d:
            tmp = os.path.join(d, "out.csv")
            _csv_write(tmp, header, cols, keep, rows, first_index, threads)
            with open(tmp) as f:
                path_or_file.write(f.read())
        return
    arr = (_lib.sf_csv_col * max(1, len(cols)))(*cols)
    L = _lib.lib()
    if L.sf_csv_write(os.fsencode(path_or_file), header.encode(), first_index, rows, len(cols), arr, threads) != 0:
        raise OSError(L.sf_csv_last_error().decode(errors="replace"))
    del keep  # the column arrays stay alive until the call has returned


def params_csv_header(P: int, flags: bool = False) -> str:
    cols = ["index", "x", "y", "sigma"] + (["sigma_y"] if P == 4 else []) + ["alpha", "beta", "status",
                                                                           "iterations", "nchi2"]
    return ",".join(cols + (["flags"] if flags else []))


def write_params_csv(path_or_file, result, first_index: int = 0, flags: bool = False, threads: int = 0) -> None:
    """ParamsCSV from a BatchResult-like object (params, alpha, beta, nchi2, status,
    iterations).  flags=True appends a `flags` column (status & 0xf8: 64 InvalidInput, 128 no-improvement)
    so assess can count the no-improvement stops (acceptance criterion 5); off by default, which keeps the
    SPEC header."""
    from . import _lib

    params = np.ascontiguousarray(result.params, np.float32)
    K = params.shape[1]
    P = 4 if K == 4 else 3  # explicit5 rows: (x, y, sigma) + alpha/beta columns
    alpha, beta, nchi2 = (np.ascontiguousarray(getattr(result, k), np.float32) for k in ("alpha", "beta", "nchi2"))
    status = np.ascontiguousarray(result.status, np.uint8)
    iters = np.ascontiguousarray(result.iterations, np.uint8)
    n = len(alpha)
    if params.shape[0] != n or len(beta) != n or len(nchi2) != n or len(status) != n or len(iters) != n:
        raise ValueError("result arrays differ in length")
    pcols = [_lib.sf_csv_col(_lib.SF_CSV_F32, params.ctypes.data + 4 * k, K) for k in range(P)]
    cols = pcols + [_col(_lib.SF_CSV_F32, alpha), _col(_lib.SF_CSV_F32, beta), _col(_lib.SF_CSV_STOP, status),
                    _col(_lib.SF_CSV_U8, iters), _col(_lib.SF_CSV_F32, nchi2)]
    if flags:
        cols.append(_col(_lib.SF_CSV_FLAGS, status))
    _csv_write(path_or_file, params_csv_header(P, flags), cols, (params, alpha, beta, nchi2, status, iters), n,
               first_index, threads)


def write_truth_csv(path_or_file, truth: np.ndarray, threads: int = 0) -> None:
    """Truth CSV: index,x,y,sigma[,sigma_y],alpha,beta."""
    from . import _lib

    truth = np.ascontiguousarray(truth, np.float32)
    K = truth.shape[1]
    names = ["x", "y", "sigma"] + (["sigma_y"] if K == 6 else []) + ["alpha", "beta"]
    if len(names) != K:
        raise ValueError(f"truth has {K} columns (5 or 6)")
    cols = [_lib.sf_csv_col(_lib.SF_CSV_F32, truth.ctypes.data + 4 * k, K) for k in range(K)]
    _csv_write(path_or_file, ",".join(["index"] + names), cols, truth, truth.shape[0], 0, threads)


def _csv_read(path: str, kinds: dict, threads: int = 0):
    """-> (index (n,), {name: array}) for the columns named in kinds (name -> (SF_CSV kind, dtype));
    other columns are skipped, a missing one raises ValueError."""
    from . import _lib

    with open(path) as f:
        header = f.readline().strip().split(",")
    if header[0] != "index":
        raise ValueError(f"{path}: header must start with 'index'")
    missing = [k for k in kinds if k not in header[1:]]
    if missing:
        raise ValueError(f"{path}: missing columns {missing}")
    L = _lib.lib()
    rows = ctypes.c_int64(0)
    if L.sf_csv_read(os.fsencode(path), ctypes.byref(rows), None, 0, None, -1, threads) != 0:  # count rows
        raise ValueError(L.sf_csv_last_error().decode(errors="replace"))
    n = rows.value
    out = {k: np.empty(n, dt) for k, (_, dt) in kinds.items()}
    index = np.empty(n, np.int64)
    cols = [_lib.sf_csv_col(kinds[h][0], out[h].ctypes.data, 1) if h in kinds else
            _lib.sf_csv_col(_lib.SF_CSV_SKIP, None, 1) for h in header[1:]]
    arr = (_lib.sf_csv_col * max(1, len(cols)))(*cols)
    if L.sf_csv_read(os.fsencode(path), ctypes.byref(rows), index.ctypes.data, len(cols), arr, n, threads) != 0:
        raise ValueError(L.sf_csv_last_error().decode(errors="replace"))
    if rows.value != n:
        raise ValueError(f"{path}: changed while reading")
    return index, out


def read_params_csv(path: str, threads: int = 0) -> dict:
    """Parse a ParamsCSV back into arrays (round trip of write_params_csv).  `flags` is
    present only when the file carries the optional flags column."""
    from . import _lib

    with open(path) as f:
        head = f.readline().strip().split(",")
    P = 4 if "sigma_y" in head else 3
    pnames = ["x", "y", "sigma"] + (["sigma_y"] if P == 4 else [])
    F32 = (_lib.SF_CSV_F32, np.float32)
    kinds = {p: F32 for p in pnames}
    kinds.update(alpha=F32, beta=F32, nchi2=F32, status=(_lib.SF_CSV_STOP, np.uint8),
                 iterations=(_lib.SF_CSV_U8, np.uint8))
    if "flags" in head:
        kinds["flags"] = (_lib.SF_CSV_FLAGS, np.uint8)
    index, c = _csv_read(path, kinds, threads)
    out = {
        "index": index,
        "params": np.stack([c[p] for p in pnames], axis=1),
        "alpha": c["alpha"], "beta": c["beta"], "nchi2": c["nchi2"], "stop": c["status"],
        "iterations": c["iterations"],
    }
    if "flags" in c:
        out["flags"] = c["flags"]
    return out


def read_truth_csv(path: str, threads: int = 0) -> np.ndarray:
    """Truth CSV -> (count, 5|6) float32 [x, y, sigma(, sigma_y), alpha, beta]."""
    from . import _lib

    with open(path) as f:
        names = f.readline().strip().split(",")[1:]
    if not names:
        raise ValueError(f"{path}: no value columns")
    _, c = _csv_read(path, {h: (_lib.SF_CSV_F32, np.float32) for h in names}, threads)
    return np.stack([c[h] for h in names], axis=1)
