"""Sharding of independent DAGs across ranks/GPUs (no collective on the data
path: DAGs are independent, experiment.cpp:56-57).

The same contiguous split as ds_analyze_batch_multi (csrc/capi.cu):
rank i of N owns DAGs [n*i/N, n*(i+1)/N).
"""
from __future__ import annotations


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return n * rank // world, n * (rank + 1) // world


def shard_seed(base_seed: int, per_rank: int, rank: int) -> int:
    """bench.py's weak-scaling shard: rank r analyses generate_corpus(seed =
    base + r * per_rank, per_rank), i.e. DAGs r*per_rank .. (r+1)*per_rank-1 of
    one global corpus."""
    return base_seed + rank * per_rank
