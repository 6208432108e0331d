"""Multi-GPU path sharding: paths are independent, so N GPUs of one node each take
a static slice of the start-index range [lo, hi) through track_all's own (lo, hi) contract,
track it to completion on their own device, and the records are gathered to rank 0 once at the
end and merged in path_id order (tracker.cpp:537-538).  There is no collective inside the
tracking loop; torch.distributed (NCCL on GPUs, gloo in the CPU tests) only moves the finished
records.
"""

from __future__ import annotations

import numpy as np

FIELDS = ("path_id", "status", "reason", "steps", "newton_iters", "rejections", "x", "residual")


def shard_range(lo: int, hi: int, rank: int, world: int) -> tuple[int, int]:
    """contiguous near-equal slice of [lo, hi) for `rank` (the first (hi-lo) % world ranks get one
    extra path); slices are disjoint and cover [lo, hi) in rank order"""
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


def distributed_track_all(track_fn, lo: int, hi: int, dist=None, group=None):
    """Run `track_fn(lo_r, hi_r) -> record dict` on this rank's slice and gather the records to
    rank 0 (None elsewhere).  Without torch.distributed it is a single-rank call."""
    if dist is None or not dist.is_initialized():
        return merge_records([track_fn(lo, hi)])
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    a, b = shard_range(lo, hi, rank, world)
    mine = track_fn(a, b) if b > a else None
    recs = {k: np.asarray(mine[k]) for k in FIELDS} if mine is not None else None
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(recs, gathered, dst=0, group=group)
    if rank != 0:
        return None
    return merge_records(gathered)
