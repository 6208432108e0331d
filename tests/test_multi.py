"""Multi-GPU sharding logic on CPU: world_size 2 over gloo.  Each rank tracks its static slice of
the start range with the C oracle standing in for its GPU, rank 0 gathers and merges; the merged
records must equal a single-process run bit for bit (paths are independent)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, read


def test_block_cyclic_shards_partition():
    from paper_1505_00383_b200.shard import contiguous_range, shard_indices, shard_size

    for lo, hi, world, block in [(0, 120, 2, 64), (5, 6, 4, 1), (0, 0, 3, 8), (100, 12345, 8, 64), (7, 19, 5, 3)]:
        parts = [shard_indices(lo, hi, r, world, block) for r in range(world)]
        assert [len(p) for p in parts] == [shard_size(lo, hi, r, world, block) for r in range(world)]
        allids = np.sort(np.concatenate(parts))
        assert np.array_equal(allids, np.arange(lo, max(lo, hi), dtype=np.uint64))
        for p in parts:
            assert np.all(np.diff(p.astype(np.int64)) > 0)
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= block
        cparts = [contiguous_range(lo, hi, r, world) for r in range(world)]
        assert cparts[0][0] == lo and cparts[-1][1] == max(lo, hi)


def test_shard_size_matches_the_library(pp):
    """pp_shard_size (C ABI) and the Python mirror agree"""
    from paper_1505_00383_b200.shard import shard_size

    for lo, hi, world, block in [(0, 120, 2, 64), (5, 6, 4, 1), (100, 12345, 8, 64), (7, 19, 5, 3), (0, 3628800, 8, 64)]:
        for r in range(world):
            assert pp.shard_size(lo, hi, (r, world, block)) == shard_size(lo, hi, r, world, block)


def test_bench_spawns_one_rank_per_gpu():
    """`bench.py --gpus 2` outside torchrun launches two ranks itself (torch.distributed.run on
    127.0.0.1); --launch-check makes each rank report its geometry without GPU work"""
    import json
    import re
    import subprocess
    import sys

    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(m) for m in re.findall(r"\{[^{}]*\}", out.stdout)]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 for d in lines)
    assert sorted(tuple(d["shard"]) for d in lines) == [(0, 2, 64), (1, 2, 64)]


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

    def fn(lo, hi, shard):
        from paper_1505_00383_b200.shard import shard_indices

        ids = shard_indices(lo, hi, *shard) if shard else np.arange(lo, hi, dtype=np.uint64)
        starts = np.stack([O.ref_td_solution(text, prec, int(i), plan["dim"]) for i in ids])
        r = O.oracle_track(plan, cfg, starts)
        r["path_id"] = ids
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
    merged = distributed_track_all(fn, 3, 120, dist, block=16)
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
