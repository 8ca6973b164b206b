"""Batch sharding across GPUs / ranks.

Spots are independent, so a batch is split into contiguous
index ranges, one per device (the C-ABI's sf_fit_batch does the same split
internally: count*d/nd .. count*(d+1)/nd).  There is no collective on the
data path; under torchrun every rank fits its own shard and only timing
plumbing crosses ranks.
"""
from __future__ import annotations


def shard_range(count: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) of `count` spots owned by `rank` of `world`
    (identical to the split in csrc/sf_capi.cu:sf_fit_batch)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return count * rank // world, count * (rank + 1) // world


def gather_results(parts: list) -> dict:
    """Concatenate per-shard result dicts in rank order (order-preserving,
    SPEC.md:384)."""
    import numpy as np

    keys = parts[0].keys()
    return {k: np.concatenate([p[k] for p in parts]) for k in keys}
