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

import io
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


def write_params_csv(path_or_file, result, first_index: int = 0) -> None:
    """ParamsCSV from a BatchResult-like object (params, alpha, beta, nchi2, status, iterations)."""
    P = min(result.params.shape[1], 4)  # explicit5 rows: (x, y, sigma) + alpha/beta columns
    if result.params.shape[1] == 5:
        P = 3
    cols = ["index", "x", "y", "sigma"] + (["sigma_y"] if P == 4 else []) + ["alpha", "beta", "status",
                                                                           "iterations", "nchi2"]
    n = len(result.alpha)
    strs = [fmt32(result.params[:, k]) for k in range(P)]
    a, b, c = fmt32(result.alpha), fmt32(result.beta), fmt32(result.nchi2)
    out = io.StringIO()
    out.write(",".join(cols) + "\n")
    for i in range(n):
        row = [str(first_index + i)] + [s[i] for s in strs] + [a[i], b[i], status_name(result.status[i]),
                                                               str(int(result.iterations[i])), c[i]]
        out.write(",".join(row) + "\n")
    _write_text(path_or_file, out.getvalue())


def write_truth_csv(path_or_file, truth: np.ndarray) -> None:
    P = truth.shape[1] - 2
    cols = ["index", "x", "y", "sigma"] + (["sigma_y"] if P == 4 else []) + ["alpha", "beta"]
    strs = [fmt32(truth[:, k]) for k in range(truth.shape[1])]
    out = io.StringIO()
    out.write(",".join(cols) + "\n")
    for i in range(truth.shape[0]):
        out.write(",".join([str(i)] + [s[i] for s in strs]) + "\n")
    _write_text(path_or_file, out.getvalue())


def _write_text(path_or_file, text: str) -> None:
    if hasattr(path_or_file, "write"):
        path_or_file.write(text)
    else:
        with open(path_or_file, "w") as f:
            f.write(text)


def read_params_csv(path: str) -> dict:
    """Parse a ParamsCSV back into arrays (round-trip of write_params_csv)."""
    with open(path) as f:
        header = f.readline().strip().split(",")
        rows = [line.rstrip("\n").split(",") for line in f if line.strip()]
    col = {h: i for i, h in enumerate(header)}
    P = 4 if "sigma_y" in col else 3
    pnames = ["x", "y", "sigma"] + (["sigma_y"] if P == 4 else [])
    n = len(rows)
    out = {
        "index": np.array([int(r[col["index"]]) for r in rows], np.int64),
        "params": np.array([[np.float32(r[col[p]]) for p in pnames] for r in rows], np.float32).reshape(n, P),
        "alpha": np.array([np.float32(r[col["alpha"]]) for r in rows], np.float32),
        "beta": np.array([np.float32(r[col["beta"]]) for r in rows], np.float32),
        "nchi2": np.array([np.float32(r[col["nchi2"]]) for r in rows], np.float32),
        "stop": np.array([STOP_NAMES.index(r[col["status"]]) for r in rows], np.uint8),
        "iterations": np.array([int(r[col["iterations"]]) for r in rows], np.uint8),
    }
    return out


def read_truth_csv(path: str) -> np.ndarray:
    with open(path) as f:
        header = f.readline().strip().split(",")
        rows = [line.rstrip("\n").split(",") for line in f if line.strip()]
    return np.array([[np.float32(v) for v in r[1:]] for r in rows], np.float32).reshape(len(rows), len(header) - 1)
