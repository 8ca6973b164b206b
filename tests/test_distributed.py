"""Multi-rank sharding on CPU (gloo, world_size 2): every rank fits its
contiguous shard (with the C oracle standing in for the device), the shards are
gathered in rank order, and the result equals the single-process batch
bit-for-bit (results independent of worker count)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import bits_equal, load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, key, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    from oracle import lm, oracle_c
    from paper_2106_02045_b200.sharding import shard_range

    fit = load_golden("fit_golden.npz")
    W, H = (int(v) for v in key.split("x"))
    im, ini = fit[f"{key}_images"], fit[f"{key}_inits"]
    lo, hi = shard_range(len(ini), rank, world)
    r = oracle_c.fit_batch(im[lo:hi], ini[lo:hi], W, H, lm.LMConfig.for_grid(W, H), threads=1)
    # gather: params as raw bytes so the comparison is bitwise
    payload = np.concatenate([r["params"].view(np.uint8).ravel(), r["status"], r["iterations"]])
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([payload.size]))
    mx = int(max(s.item() for s in sizes))
    buf = torch.zeros(mx, dtype=torch.uint8)
    buf[: payload.size] = torch.from_numpy(payload)
    bufs = [torch.zeros(mx, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(bufs, buf)
    # max-over-ranks timing plumbing, as bench.py does
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        parts = []
        for rk, (b, s) in enumerate(zip(bufs, sizes)):
            a, c = shard_range(len(ini), rk, world)
            n = c - a
            raw = b[: int(s.item())].numpy()
            parts.append(dict(params=raw[: n * 12].view(np.float32).reshape(n, 3), status=raw[n * 12: n * 13],
                              iterations=raw[n * 13: n * 14]))
        from paper_2106_02045_b200.sharding import gather_results

        g = gather_results(parts)
        np.savez(os.path.join(out_dir, "gathered.npz"), **g, tmax=t.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("key", ["15x15", "11x11"])
def test_two_rank_shards_equal_single_process(tmp_path, key):
    world = 2
    mp.spawn(_rank_main, args=(world, _free_port(), key, str(tmp_path)), nprocs=world, join=True)
    g = np.load(tmp_path / "gathered.npz")
    fit = load_golden("fit_golden.npz")
    assert bits_equal(g["params"], fit[f"{key}_params"])
    assert np.array_equal(g["status"], fit[f"{key}_status"])
    assert np.array_equal(g["iterations"], fit[f"{key}_iterations"])
    assert float(g["tmax"][0]) == 2.0


def test_shard_range_partition():
    from paper_2106_02045_b200.sharding import shard_range

    for count in (0, 1, 7, 1000, 10**8):
        for world in (1, 2, 3, 8):
            rs = [shard_range(count, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1


def _gpu_rank_main(rank, world, port, out_dir):
    """One torchrun-style rank on the product path: fit_shard on this rank's device (all ranks share
    cuda:0 on a one-GPU box), gather the shards over gloo in rank order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    import paper_2106_02045_b200 as sf
    from paper_2106_02045_b200.sharding import fit_shard

    W = H = 15
    im, _ = sf.simulate_batch(sf.SimConfig(width=W, height=H, count=5003, seed=61))
    lo, hi, r = fit_shard(im, None, rank=rank, world=world, device=0)
    payload = np.concatenate([r.params.view(np.uint8).ravel(), r.alpha.view(np.uint8), r.status, r.iterations])
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([payload.size]))
    mx = int(max(s.item() for s in sizes))
    buf = torch.zeros(mx, dtype=torch.uint8)
    buf[: payload.size] = torch.from_numpy(payload)
    bufs = [torch.zeros(mx, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(bufs, buf)
    if rank == 0:
        from paper_2106_02045_b200.sharding import gather_results, shard_range

        parts = []
        for rk, (b, s) in enumerate(zip(bufs, sizes)):
            a, c = shard_range(len(im), rk, world)
            n = c - a
            raw = b[: int(s.item())].numpy()
            parts.append(dict(params=raw[: n * 12].view(np.float32).reshape(n, 3),
                              alpha=raw[n * 12: n * 16].view(np.float32), status=raw[n * 16: n * 17],
                              iterations=raw[n * 17: n * 18]))
        g = gather_results(parts)
        whole = sf.fit_batch(im)
        np.savez(os.path.join(out_dir, "gpu_gathered.npz"), **g, w_params=whole.params, w_alpha=whole.alpha,
                 w_status=whole.status, w_iterations=whole.iterations)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_product_shards_equal_whole_batch(tmp_path):
    """The product's multi-rank path (fit_shard = sf_shard_range + fit_batch on the rank's device, the
    fused initializer inside each shard) gathered over gloo equals one fit_batch of the whole batch."""
    world = 2
    mp.spawn(_gpu_rank_main, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g = np.load(tmp_path / "gpu_gathered.npz")
    assert bits_equal(g["params"], g["w_params"]) and bits_equal(g["alpha"], g["w_alpha"])
    assert np.array_equal(g["status"], g["w_status"]) and np.array_equal(g["iterations"], g["w_iterations"])


def test_library_shard_split_matches_formula():
    from paper_2106_02045_b200.sharding import shard_range

    for count in (0, 5, 10**8, 2**62):
        for world in (1, 3, 8, 1000):
            for r in (0, world // 2, world - 1):
                assert shard_range(count, r, world) == (count * r // world, count * (r + 1) // world)
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
