"""Multi-GPU sharding logic on CPU: world_size 2 over gloo.  Each rank tracks its static slice of
the start range with the C oracle standing in for its GPU, rank 0 gathers and merges; the merged
records must equal a single-process run bit for bit (paths are independent)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, read


def test_shard_range_partitions():
    from paper_1505_00383_b200.shard import shard_range

    for lo, hi, world in [(0, 120, 2), (5, 6, 4), (0, 0, 3), (100, 1234567, 8), (7, 19, 5)]:
        parts = [shard_range(lo, hi, r, world) for r in range(world)]
        assert parts[0][0] == lo and parts[-1][1] == max(lo, hi)
        for (a, b), (c, d) in zip(parts, parts[1:]):
            assert b == c
        sizes = [b - a for a, b in parts]
        assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_track_fn(text, prec):
    import oracle as O

    gam = O.ref_random_gamma(1)
    L = O.LIMBS[prec]
    gl = np.zeros(2 * L)
    gl[0], gl[L] = gam.real, gam.imag
    plan = O.ref_plan(text, prec, gl)
    cfg = O.ref_defaults(prec)

    def fn(lo, hi):
        starts = np.stack([O.ref_td_solution(text, prec, i, plan["dim"]) for i in range(lo, hi)])
        r = O.oracle_track(plan, cfg, starts)
        r["path_id"] = np.arange(lo, hi, dtype=np.uint64)
        return r

    return fn


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1505_00383_b200.shard import distributed_track_all

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fn = _oracle_track_fn(read("cyclic5.sys"), "d")
    merged = distributed_track_all(fn, 3, 120, dist)
    if rank == 0:
        np.savez(os.path.join(out_dir, "merged.npz"), **merged)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_equals_single_process(tmp_path, oracle_mod):
    if oracle_mod.ref is None:
        pytest.skip("reference build not present")
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    with np.load(tmp_path / "merged.npz") as z:
        merged = {k: z[k] for k in z.files}
    from conftest import golden

    g = golden("track_cyclic5_d")
    assert np.array_equal(merged["path_id"], np.arange(3, 120, dtype=np.uint64))
    for k in ("status", "reason", "steps", "newton_iters", "rejections", "x", "residual"):
        assert np.array_equal(merged[k], g[k][3:]), k
