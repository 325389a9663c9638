"""N>1 host-side logic with world_size-2 gloo process groups on CPU.

The data path has no collective (DAGs are independent); what must hold is
that per-rank shards partition the corpus, that gathering per-rank results
in rank order reproduces the single-process results (checked with the CPU
oracle standing in for each rank's device), and that the timing reduction
bench.py uses (all_reduce MAX) yields the slowest rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_20826_b200.shard import shard_bounds, shard_seed


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.bindings import Checker
    orc = Checker("oracle")
    # (1) shard of a global corpus, as ds_analyze_batch_multi splits it
    full = orc.generate(n, seed=1).pack()
    from paper_2602_20826_b200 import _lib
    lo, hi = _lib.shard_range(n, world, rank)  # the split capi.cu's multi entry points use
    assert (lo, hi) == shard_bounds(n, world, rank)
    st, b, _ = orc.corpus(full.slice(lo, hi)).evaluate(148)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([hi - lo]))
    mx = max(int(s) for s in sizes)
    pad = torch.zeros((mx, 10), dtype=torch.int64)
    pad[:hi - lo] = torch.from_numpy(b)
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    # (2) weak-scaling shard by seed (bench.py)
    per = n // world
    own = orc.generate(per, seed=shard_seed(1, per, rank)).pack()
    st2, b2, _ = orc.corpus(own).evaluate(148)
    bufs2 = [torch.zeros((per, 10), dtype=torch.int64) for _ in range(world)]
    dist.all_gather(bufs2, torch.from_numpy(b2))
    # (3) max-over-ranks timing
    t = torch.tensor([float(rank + 1) * 1.5], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        gathered = np.concatenate([bufs[r][:int(sizes[r])].numpy() for r in range(world)])
        np.save(os.path.join(out_dir, "gathered.npy"), gathered)
        np.save(os.path.join(out_dir, "weak.npy"), np.concatenate([x.numpy() for x in bufs2]))
        np.save(os.path.join(out_dir, "tmax.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds_partition():
    for n in (0, 1, 7, 1000, 1_000_003):
        for world in (1, 2, 3, 8):
            edges = [shard_bounds(n, world, r) for r in range(world)]
            assert edges[0][0] == 0 and edges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(edges, edges[1:]))
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_library_split_equals_shard_py():
    """ds_shard_range (the split of ds_analyze_batch[16]_multi, capi.cu) is
    shard.py's split for every rank, including n not divisible by N and
    n < N, and rejects a bad shard index."""
    from paper_2602_20826_b200 import _lib
    for n in (0, 1, 5, 7, 1000, 1_000_003, 2**40 + 17):
        for world in (1, 2, 3, 7, 8):
            for r in range(world):
                assert _lib.shard_range(n, world, r) == shard_bounds(n, world, r)
    with pytest.raises(_lib.DagschedError):
        _lib.shard_range(10, 2, 2)


def test_world2_gloo_shards_reproduce_single_process(tmp_path):
    world, n = 2, 600
    mp.spawn(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True)
    from oracle.bindings import Checker
    orc = Checker("oracle")
    _, ref, _ = orc.generate(n, seed=1).evaluate(148)
    assert np.array_equal(np.load(tmp_path / "gathered.npy"), ref)
    # shards by seed are the slices of one global corpus
    assert np.array_equal(np.load(tmp_path / "weak.npy"), ref[:n // world * world])
    assert float(np.load(tmp_path / "tmax.npy")[0]) == 3.0
