"""The production engine against the reference, and the boundary's optional arguments.

* Production occupancy: one benchmark-sized call (all slots, TMEM evaluation, refill, tail
  compaction, CUDA graphs, tail mode) at default knobs, its records checked bit for bit against
  reference records of eight ranges spread over the call (tests/golden/make_golden_prod.py).
* Shards (pp_shard): block-cyclic partitions of a range reproduce the unsharded records.
* Step events (ProgressSink, tracker.hpp:62-70): per path, the device's events equal the
  reference sink's (tracker.cpp:312-315), field for field and in order."""

import numpy as np
import pytest

from conftest import golden, read
from test_gpu_parity import TRACK_KEYS, bits, homotopy

pytestmark = pytest.mark.gpu


def assert_golden_ranges(sol, g, call_lo):
    per = int(g["range_len"])
    for i, a in enumerate(g["range_lo"]):
        off = int(a) - call_lo
        for k in TRACK_KEYS:
            got = bits(getattr(sol, k)[off:off + per])
            want = bits(g[k][i * per:(i + 1) * per])
            assert np.array_equal(got, want), (k, int(a))
        assert np.array_equal(sol.path_id[off:off + per], g["path_id"][i * per:(i + 1) * per])


@pytest.mark.parametrize("name,plain", [("cyclic10_dd_prod", False), ("cyclic10_d_prod", False),
                                        ("cyclic10_dd_prod", True)])
def test_production_occupancy_bitwise(pp, monkeypatch, name, plain):
    """BASELINE config 3 at the bench's size: cyclic-10 dd over 262,144 paths (592 blocks of 128
    slots, open row in TMEM, 16-trip graphs, compaction, tail mode); cyclic-10 d over 524,288 paths
    (1,024 slots per SM, register-resident solver)"""
    if plain:  # the round-1 solver: shared-memory column, no TMEM q-cache
        monkeypatch.setenv("PP200_LSQ_QCACHE", "0")
    g = golden(f"track_{name}")
    prec = str(g["prec"])
    _, _, starts, h = homotopy(pp, read("cyclic10.sys"), prec)
    lo, hi = int(g["call_lo"]), int(g["call_hi"])
    sol = pp.track_all(h, starts, lo=lo, hi=hi)
    assert len(sol) == hi - lo
    assert np.array_equal(sol.path_id, np.arange(lo, hi, dtype=np.uint64))
    assert np.all((sol.status == pp.SUCCESS) | (sol.status == pp.FAILED))
    assert sol.stats["slots"] == (75_776 if prec == "dd" else 151_552)
    assert_golden_ranges(sol, g, lo)
    # the far golden range of round 1 lies inside the dd call as well
    if prec == "dd":
        far = golden("track_cyclic10_dd_far")
        a = int(far["lo"]) - lo
        for k in TRACK_KEYS:
            assert np.array_equal(bits(getattr(sol, k)[a:a + 32]), bits(far[k])), k


@pytest.mark.parametrize("system,prec,lo,hi,block,nshard", [
    ("cyclic5", "d", 0, 120, 7, 3), ("cyclic5", "dd", 3, 120, 16, 4), ("cyclic10", "d", 0, 512, 64, 8),
])
def test_shards_reproduce_the_range(pp, system, prec, lo, hi, block, nshard):
    g = golden(f"track_{system}_{prec}")
    _, _, starts, h = homotopy(pp, read(f"{system}.sys"), prec)
    parts = []
    for r in range(nshard):
        sol = pp.track_all(h, starts, lo=lo, hi=hi, shard=(r, nshard, block))
        assert len(sol) == pp.shard_size(lo, hi, (r, nshard, block))
        ids = np.arange(lo, hi)
        assert np.array_equal(sol.path_id, ids[((ids - lo) // block) % nshard == r])
        parts.append(sol)
    ids = np.concatenate([p.path_id for p in parts])
    order = np.argsort(ids, kind="stable")
    assert np.array_equal(ids[order], np.arange(lo, hi, dtype=np.uint64))
    for k in TRACK_KEYS:
        merged = np.concatenate([getattr(p, k) for p in parts])[order]
        assert np.array_equal(bits(merged), bits(g[k][lo - int(g["lo"]):hi - int(g["lo"])])), k


def per_path(ev):
    """events grouped by path, each path's events in emission order"""
    order = np.argsort(ev["path_id"], kind="stable")
    return ev[order]


@pytest.mark.parametrize("name", ["cyclic5_d", "cyclic5_dd", "cyclic5_d_tight"])
@pytest.mark.parametrize("mode", ["default", "thread_per_path", "warp_per_path", "group8_per_path"])
def test_step_events_match_the_reference_sink(pp, monkeypatch, name, mode):
    g = golden(f"events_{name}")
    prec = str(g["prec"])
    if mode.startswith("thread_per_path"):
        monkeypatch.setenv("PP200_TAIL_SLOTS", "0")
        monkeypatch.setenv("PP200_COOP_WHOLE_RUN", "0")
    elif mode == "group8_per_path":
        monkeypatch.setenv("PP200_FORCE_COOP", "1")
        monkeypatch.setenv("PP200_COOP_GROUP", "8")
        monkeypatch.setenv("PP200_COOP_GROUP_EVAL", "8")
    elif mode == "warp_per_path":
        monkeypatch.setenv("PP200_FORCE_COOP", "1")
    _, _, starts, h = homotopy(pp, read("cyclic5.sys"), prec)
    cfg = pp.TrackConfig.defaults(prec)
    for k, v in eval(str(g["cfg"])).items():
        setattr(cfg, k, v)
    got = []
    sol = pp.track_all(h, starts, cfg, lo=int(g["lo"]), hi=int(g["hi"]), sink=got.append)
    ev = np.concatenate(got)
    want = g["events"]
    assert sol.stats["events"] == len(ev) == len(want)
    a, b = per_path(ev), per_path(want)
    for f in ("path_id", "newton_iters", "status", "accepted"):
        assert np.array_equal(a[f], b[f]), f
    for f in ("t", "h"):
        assert np.array_equal(a[f].view(np.uint64), b[f].view(np.uint64)), f
    assert np.all(a["status"] == pp.ACTIVE)
    # per path: accepted steps and rejections add up to the record's counters
    acc = np.bincount(ev["path_id"].astype(np.int64), weights=ev["accepted"], minlength=120)
    assert np.array_equal(acc.astype(np.uint32), sol.steps)
    # the records are the same with and without a sink
    for k in TRACK_KEYS:
        assert np.array_equal(bits(getattr(sol, k)), bits(g[k])), k


def test_sink_exceptions_propagate(pp):
    _, _, starts, h = homotopy(pp, read("cyclic5.sys"), "d")

    def bad(_ev):
        raise KeyError("stop")

    with pytest.raises(KeyError):
        pp.track_all(h, starts, lo=0, hi=8, sink=bad)


def test_two_ranks_share_the_gpu(tmp_path):
    """the multi-GPU path with the CUDA library: two torchrun ranks (sharing this GPU over gloo
    when the box has one) track their block-cyclic shards, rank 0 gathers and merges; the merged
    records equal the reference's"""
    import os
    import socket
    import subprocess
    import sys

    from conftest import ROOT

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "merged.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "scripts", "multi_rank_check.py"), "cyclic10",
           "d", "0", "512", "64", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    g = golden("track_cyclic10_d")
    with np.load(out) as z:
        assert np.array_equal(z["path_id"], np.arange(0, 512, dtype=np.uint64))
        for k in TRACK_KEYS:
            assert np.array_equal(bits(z[k]), bits(g[k])), k


def newton_cases():
    import os

    from conftest import GOLDEN

    z = np.load(os.path.join(GOLDEN, "newton_cases.npz"))
    return [str(n) for n in z["names"]], z


@pytest.mark.parametrize("name", newton_cases()[0])
def test_corrector_alone_matches_set_prediction(pp, name):
    """PathBatch::set_prediction + newton_correct (tracker.hpp:135-136; test_tracker.cpp:121-196,
    acceptance criterion 9): on-path, nearby, hopeless and rank-deficient predictions give the
    reference's iteration counts, certification flags and last iterates, bit for bit; the square
    homotopy reproduces the reference tests' expectations (one iteration on the path, 2.1 -> 2 in
    three, the lockstep pattern (3, 1, 2), no convergence from (250, 40) with max_newton = 2)"""
    _, z = newton_cases()
    g = {k.split("__", 1)[1]: z[k] for k in z.files if k.startswith(name + "__")}
    prec = str(g["prec"])
    L = pp.LIMBS[prec]
    f = pp.parse_system(str(g["f"]))
    gs = pp.parse_system(str(g["g"])) if str(g["g"]) else pp.total_degree_start(f, prec)[0]
    gam = complex(g["gamma"][0], g["gamma"][L])
    h = pp.make_homotopy(f, gs, gam, prec)
    cfg = pp.TrackConfig.defaults(prec)
    for k, v in eval(str(g["cfg"])).items():
        setattr(cfg, k, v)
    it, co, sg, xo = pp.newton_correct(h, g["t"], g["x"], cfg)
    assert np.array_equal(it, g["iters"])
    assert np.array_equal(co, g["corrected"])
    assert np.array_equal(bits(xo), bits(g["x_out"]))
    if name == "square_d":
        assert it.tolist()[:2] == [1, 3] and it.tolist()[4:] == [3, 1, 2] and co[0] and co[2]
    if name.startswith("cyclic"):
        assert sg[-1] and it[-1] == 1  # the origin: rank-deficient Jacobian, the solve fails at once
