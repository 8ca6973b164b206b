"""Batch sharding across GPUs / ranks.

Spots are independent, so a batch is split into contiguous, order-preserving
index ranges.  The split is the library's (sf_shard_range): sf_fit_batch
applies it over its devices inside one process (one host thread per device),
and a torchrun rank applies it over the job with fit_shard below.  No
collective touches the data path; only timing plumbing and, if the caller
wants the whole result on one rank, the final gather cross ranks.
"""
from __future__ import annotations

import ctypes

from . import _lib


def shard_range(count: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) of `count` spots owned by shard `rank` of `world` (sf_shard_range)."""
    lo, hi = ctypes.c_int64(0), ctypes.c_int64(0)
    if _lib.lib().sf_shard_range(count, rank, world, ctypes.byref(lo), ctypes.byref(hi)) != 0:
        raise ValueError(f"bad shard arguments: count={count} rank={rank} world={world}")
    return lo.value, hi.value


def fit_shard(images, inits=None, rank: int = 0, world: int = 1, device: int = 0, **kw):
    """Fit this rank's shard of `images` (count, H, W) on `device`: -> (lo, hi, BatchResult).
    Under torchrun: rank = RANK, world = WORLD_SIZE, device = LOCAL_RANK."""
    from .batch_engine import fit_batch

    lo, hi = shard_range(len(images), rank, world)
    part_inits = None if inits is None else inits[lo:hi]
    return lo, hi, fit_batch(images[lo:hi], part_inits, devices=[device], **kw)


def gather_results(parts: list) -> dict:
    """Concatenate per-shard result dicts in rank order (order-preserving)."""
    import numpy as np

    keys = parts[0].keys()
    return {k: np.concatenate([p[k] for p in parts]) for k in keys}
