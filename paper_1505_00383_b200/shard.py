"""Multi-GPU path sharding: paths are independent, so N GPUs of one node each take
a static shard of the start-index range [lo, hi) and track it to completion on their own device;
the records are gathered to rank 0 once at the end and merged in path_id order
(tracker.cpp:537-538).  There is no collective inside the tracking loop; torch.distributed (NCCL
on GPUs, gloo in the CPU tests) only moves the finished records.

Shards are block-cyclic (pp_shard in include/pp200.h): start index i belongs to shard
((i - lo) // block) % world.  Per-path cost varies strongly with the start index (cyclic-10:
[0, 128) and [1e6, 1e6 + 128) converge 19 vs 1 paths), so contiguous slices leave
some GPUs with far more work than others; interleaving small blocks evens the shards out while
each shard's device call still sees long runs of consecutive indices.
"""

from __future__ import annotations

import numpy as np

FIELDS = ("path_id", "status", "reason", "steps", "newton_iters", "rejections", "x", "residual")
DEFAULT_BLOCK = 64


def shard_indices(lo: int, hi: int, rank: int, world: int, block: int = DEFAULT_BLOCK) -> np.ndarray:
    """the start indices of [lo, hi) in block-cyclic shard `rank` of `world`, increasing (the order
    pp_track_all_ex writes its records in)"""
    ids = np.arange(lo, max(lo, hi), dtype=np.uint64)
    if world <= 1:
        return ids
    return ids[((ids - lo) // block) % world == rank]


def shard_size(lo: int, hi: int, rank: int, world: int, block: int = DEFAULT_BLOCK) -> int:
    """pp_shard_size: full block groups plus this shard's part of the remainder"""
    total = max(0, hi - lo)
    if world <= 1:
        return total
    span = block * world
    full, rem = divmod(total, span)
    first = rank * block
    return full * block + (min(block, rem - first) if rem > first else 0)


def contiguous_range(lo: int, hi: int, rank: int, world: int) -> tuple[int, int]:
    """contiguous near-equal slice of [lo, hi) (the reference CLI's --path-range partition, kept
    for the load-balance comparison in scripts/shard_balance.py)"""
    n = max(0, hi - lo)
    base, extra = divmod(n, world)
    start = lo + rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def merge_records(parts: list[dict]) -> dict:
    """concatenate per-rank record dicts and sort by path_id"""
    parts = [p for p in parts if p is not None and len(p["path_id"])]
    if not parts:
        return {}
    out = {k: np.concatenate([p[k] for p in parts]) for k in FIELDS}
    order = np.argsort(out["path_id"], kind="stable")
    return {k: v[order] for k, v in out.items()}


def distributed_track_all(track_fn, lo: int, hi: int, dist=None, group=None, block: int = DEFAULT_BLOCK):
    """Run `track_fn(lo, hi, shard) -> record dict` for this rank's block-cyclic shard
    (shard = (rank, world, block), None for a single rank) and gather the records to rank 0
    (None elsewhere), merged in path_id order."""
    if dist is None or not dist.is_initialized():
        return merge_records([track_fn(lo, hi, None)])
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = track_fn(lo, hi, (rank, world, block)) if shard_size(lo, hi, rank, world, block) else None
    recs = {k: np.asarray(mine[k]) for k in FIELDS} if mine is not None else None
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(recs, gathered, dst=0, group=group)
    if rank != 0:
        return None
    return merge_records(gathered)
