"""Parity of the CUDA path (through the C ABI) with the reference tracker.

Bit-exact against the golden records of the unmodified reference build (tests/golden) at sizes
the reference finishes in seconds; at larger sizes through size-independent properties
(determinism, scheduling invariance, range partition invariance, the convergence certificate
re-evaluated on the device, gamma independence of the endpoint set)."""

import os

import numpy as np
import pytest

from conftest import golden, read

pytestmark = pytest.mark.gpu

TRACK_KEYS = ["status", "reason", "steps", "newton_iters", "rejections", "x", "residual"]
SQUARE_F = "1; x0^2 - 4;"
SQUARE_G = "1; x0^2 - 1;"


def homotopy(P, text, prec, seed=1, g_text=None):
    f = P.parse_system(text)
    if g_text is None:
        g, starts = P.total_degree_start(f, prec)
    else:
        g, starts = P.parse_system(g_text), None
    return f, g, starts, P.make_homotopy(f, g, P.random_gamma(seed), prec)


def bits(a):
    """bit patterns of a record array (floats compared bit for bit: -0.0 differs from 0.0)"""
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


def assert_records(sol, g, lo=0):
    assert np.array_equal(sol.path_id, np.arange(lo, lo + len(sol), dtype=np.uint64))
    for k in TRACK_KEYS:
        got, want = bits(getattr(sol, k)), bits(g[k])
        if not np.array_equal(got, want):
            bad = np.flatnonzero(np.any(np.asarray(got).reshape(len(sol), -1) != np.asarray(want).reshape(len(sol), -1), axis=1))
            raise AssertionError(f"{k} differs on {len(bad)} paths, first {bad[:5]}")


# ---------------------------------------------------------------------------------------------
# kernel-level boundary: eval_system_batch and least_squares_solve
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("prec", ["d", "dd", "qd"])
@pytest.mark.parametrize("system", ["cyclic5", "cyclic10"])
def test_eval_bitwise(pp, prec, system):
    g = golden(f"eval_{system}_{prec}")
    f, gs, _, h = homotopy(pp, read(f"{system}.sys"), prec)
    sys_, jac = pp.eval_batch(h, g["points"], g["t"])
    assert np.array_equal(sys_, g["sys"])
    assert np.array_equal(jac, g["jac"])


def test_bench_eval_checksums(pp):
    """bench-eval on the device reproduces the reference's checksum (tests/golden/bench_eval.json:
    the CLI's point stream, the reference eval_system_batch, FNV-1a over the planar workspace)"""
    import json

    with open(os.path.join(os.path.dirname(__file__), "golden", "bench_eval.json")) as fh:
        cases = json.load(fh)
    for c in cases:
        _, _, _, h = homotopy(pp, read(c["system"] + ".sys"), c["prec"], seed=c["gamma_seed"])
        ms, cs = pp.bench_eval(h, c["seed"], c["batch"], reps=3)
        assert cs == c["checksum"], c
        assert ms > 0


@pytest.mark.parametrize("prec", ["d", "dd", "qd"])
@pytest.mark.parametrize("n", [1, 5, 10, 13])
def test_lsq_bitwise(pp, prec, n):
    g = golden(f"lsq_n{n}_{prec}")
    x, ok = pp.lsq_batch(prec, g["a"], g["b"])
    assert np.array_equal(ok, g["ok"].astype(bool))
    assert np.array_equal(x[ok], g["x"][ok])


# ---------------------------------------------------------------------------------------------
# track_all: bitwise against the reference records
# ---------------------------------------------------------------------------------------------
def system_text(pp, system):
    if system == "cyclic8":
        return pp.cyclic_system(8).text()
    return read(f"{system}.sys")


@pytest.mark.parametrize("name,system", [
    ("cyclic5_d", "cyclic5"), ("cyclic5_dd", "cyclic5"), ("cyclic5_qd", "cyclic5"), ("cyclic10_d", "cyclic10"),
    ("cyclic10_dd", "cyclic10"), ("cyclic10_dd_far", "cyclic10"), ("cyclic5_dd_seed101", "cyclic5"),
    ("cyclic8_d", "cyclic8"), ("cyclic8_dd", "cyclic8"), ("katsura12_d", "katsura12"),
    ("katsura12_dd", "katsura12"), ("katsura12_qd_mn4", "katsura12"), ("rand32_d", "rand32"),
    ("rand32_dd", "rand32"), ("rand32_qd", "rand32"), ("cyclic8_qd", "cyclic8"), ("cyclic10_qd", "cyclic10"),
])
def test_track_bitwise(pp, name, system):
    g = golden(f"track_{name}")
    prec = str(g["prec"])
    _, _, starts, h = homotopy(pp, system_text(pp, system), prec, seed=int(g["gamma_seed"]))
    lo, hi = int(g["lo"]), int(g["hi"])
    cfg = pp.TrackConfig.defaults(prec)
    for k, v in eval(str(g["cfg"])).items():
        setattr(cfg, k, v)
    sol = pp.track_all(h, starts, cfg, lo=lo, hi=hi)
    assert_records(sol, g, lo)


@pytest.mark.parametrize("name,system", [
    ("cyclic5_d", "cyclic5"), ("cyclic5_dd", "cyclic5"), ("cyclic5_qd", "cyclic5"), ("cyclic10_dd", "cyclic10"),
    ("katsura12_qd_mn4", "katsura12"), ("rand32_dd", "rand32"), ("cyclic8_d", "cyclic8"),
])
@pytest.mark.parametrize("mode", ["warp_per_path", "group8_per_path", "group4_per_path", "thread_per_path",
                                  "thread_per_path_tmem", "thread_per_path_plain", "thread_per_path_fuse",
                                  "thread_per_path_staged", "thread_per_path_l2hint"])
def test_track_bitwise_modes(pp, monkeypatch, name, system, mode):
    """every engine gives the reference records: every trip in tail mode (a warp per path, or 8
    or 4 lanes per path: eval_coop / lsq_coop), or never (a thread per path; small runs otherwise
    start in tail mode), also with the open Jacobian row and the Gram-Schmidt column in tensor
    memory, and without the TMEM q-cache / register-resident solvers (plain shared-memory column)"""
    if mode.endswith("_per_path") and not mode.startswith("thread"):
        monkeypatch.setenv("PP200_FORCE_COOP", "1")
        g = {"warp": "32", "group8": "8", "group4": "4"}[mode.split("_")[0]]
        monkeypatch.setenv("PP200_COOP_GROUP", g)
        monkeypatch.setenv("PP200_COOP_GROUP_EVAL", g)
    else:
        monkeypatch.setenv("PP200_TAIL_SLOTS", "0")
        monkeypatch.setenv("PP200_COOP_WHOLE_RUN", "0")
    if mode.endswith("plain"):
        monkeypatch.setenv("PP200_LSQ_QCACHE", "0")
        monkeypatch.setenv("PP200_LSQ_REG", "0")
    monkeypatch.setenv("PP200_LSQ_FUSE", "1" if mode.endswith("fuse") else "0")
    monkeypatch.setenv("PP200_LSQ_L2HINT", "1" if mode.endswith("l2hint") else "0")
    # plan tables staged in shared memory by TMA bulk copies (the default) or read from global memory
    monkeypatch.setenv("PP200_STAGE_TABLES", "1" if mode.endswith("staged") else "0")
    if mode.endswith("staged"):
        monkeypatch.setenv("PP200_TMEM", "1")
    if mode.endswith("tmem"):
        monkeypatch.setenv("PP200_TMEM", "1")
        monkeypatch.setenv("PP200_LSQ_TMEM", "1")
    else:
        monkeypatch.setenv("PP200_TMEM", "0")
    test_track_bitwise(pp, name, system)


def test_track_custom_config_bitwise(pp):
    """non-default TrackConfig (failure-heavy): max_newton 2, h_init 0.1, max_steps 40"""
    g = golden("track_cyclic5_d_tight")
    _, _, starts, h = homotopy(pp, read("cyclic5.sys"), "d")
    cfg = pp.TrackConfig.defaults("d")
    cfg.max_newton, cfg.h_init, cfg.max_steps = 2, 0.1, 40
    sol = pp.track_all(h, starts, cfg)
    assert_records(sol, g)
    assert set(pp.REASONS[r] for r in sol.reason[sol.status == pp.FAILED]) >= {"max-steps"}


def test_track_square_explicit_starts(pp):
    g = golden("track_square_d")
    f, gs, _, h = homotopy(pp, SQUARE_F, "d", g_text=SQUARE_G)
    starts = pp.explicit_starts(np.array([[[1.0, 0.0]], [[-1.0, 0.0]]]), "d")
    sol = pp.track_all(h, starts)
    assert_records(sol, g)


def test_track_cyclic3_dd(pp):
    g = golden("track_cyclic3_dd")
    _, _, starts, h = homotopy(pp, pp.cyclic_system(3).text(), "dd", seed=3)
    assert_records(pp.track_all(h, starts), g)


def test_track_from_start_file(pp):
    """the `polypath track` entry: user start system + start file through load_start_data"""
    g = golden("track_cyclic5_file_dd")
    f = pp.parse_system(read("cyclic5.sys"))
    gs = pp.parse_system(read("cyclic5_start.sys"))
    starts, rejected = pp.load_start_data(gs, read("cyclic5_starts.txt"), "dd")
    assert rejected == [] and starts.count == 120
    h = pp.make_homotopy(f, gs, pp.random_gamma(1), "dd")
    assert_records(pp.track_all(h, starts), g)


def test_load_start_data_rejects_bad_candidates(pp):
    gs = pp.parse_system("2; x0^2 - 1; x1 - 1;")
    text = "1,0, 1,0\n-1,0, 1,0\n0.5,0, 1,0\n(1,1e-12),(1,0)\n"
    starts, rejected = pp.load_start_data(gs, text, "dd")
    assert starts.count == 3
    assert [i for i, _ in rejected] == [2] and abs(rejected[0][1] - 0.75) < 1e-15


# ---------------------------------------------------------------------------------------------
# edge cases of the boundary (tracker.cpp:511-540)
# ---------------------------------------------------------------------------------------------
def test_ranges_and_errors(pp):
    _, _, starts, h = homotopy(pp, read("cyclic5.sys"), "d")
    g = golden("track_cyclic5_d")
    assert len(pp.track_all(h, starts, lo=50, hi=50)) == 0           # empty range
    assert len(pp.track_all(h, starts, lo=130, hi=140)) == 0         # beyond the start set
    sol = pp.track_all(h, starts, lo=117, hi=10_000)                 # clipped to count
    assert len(sol) == 3
    assert np.array_equal(sol.x, g["x"][117:])
    one = pp.track_all(h, starts, lo=7, hi=8)                          # a single path
    assert np.array_equal(one.x[0], g["x"][7])
    bad = pp.TrackConfig.defaults("d")
    bad.h_min = 0.5
    with pytest.raises(pp.InvalidArgument):
        pp.track_all(h, starts, bad)
    empty = pp.explicit_starts(np.zeros((0, 5, 2)), "d")
    with pytest.raises(pp.InvalidArgument):
        pp.track_all(h, empty)


# ---------------------------------------------------------------------------------------------
# properties at larger sizes
# ---------------------------------------------------------------------------------------------
def test_cyclic10_dd_properties(pp, monkeypatch):
    """16384 paths far into the index space: terminal statuses, certificate re-checked on the
    device, determinism, and invariance under slot count and range partition."""
    _, _, starts, h = homotopy(pp, read("cyclic10.sys"), "dd")
    lo, hi = 2_000_000, 2_016_384
    a = pp.track_all(h, starts, lo=lo, hi=hi)
    assert np.all((a.status == pp.SUCCESS) | (a.status == pp.FAILED))
    rtol = pp.TrackConfig.defaults("dd").residual_tol
    ok = a.status == pp.SUCCESS
    res = a.residual[:, 0] + a.residual[:, 1]
    assert np.all(res[ok] <= 10 * rtol)
    # certificate: |f(x)| at the endpoint re-evaluated by the device equals the record residual
    t1 = np.zeros((int(ok.sum()), 2))
    t1[:, 0] = 1.0
    sys_, _ = pp.eval_batch(h, a.x[ok], t1)
    m = np.sqrt(sys_[..., 0] ** 2 + sys_[..., 2] ** 2).max(axis=1)
    assert np.allclose(m, res[ok], rtol=1e-6, atol=1e-30)
    # determinism and scheduling invariance
    b = pp.track_all(h, starts, lo=lo, hi=hi)
    monkeypatch.setenv("PP200_SLOTS_PER_SM", "128")
    monkeypatch.setenv("PP200_GRAPH_TRIPS", "3")
    monkeypatch.setenv("PP200_COMPACT", "0")
    c = pp.track_all(h, starts, lo=lo, hi=hi)
    monkeypatch.delenv("PP200_SLOTS_PER_SM")
    monkeypatch.delenv("PP200_GRAPH_TRIPS")
    monkeypatch.delenv("PP200_COMPACT")
    monkeypatch.setenv("PP200_KERNEL_TIMING", "1")  # per-trip launches, compaction between trips
    e = pp.track_all(h, starts, lo=lo, hi=hi)
    monkeypatch.delenv("PP200_KERNEL_TIMING")
    mid = lo + 5000
    d1 = pp.track_all(h, starts, lo=lo, hi=mid)
    d2 = pp.track_all(h, starts, lo=mid, hi=hi)
    for k in TRACK_KEYS:
        ref = getattr(a, k)
        assert np.array_equal(ref, getattr(b, k)), k
        assert np.array_equal(ref, getattr(c, k)), k
        assert np.array_equal(ref, getattr(e, k)), k
        assert np.array_equal(ref, np.concatenate([getattr(d1, k), getattr(d2, k)])), k


def test_gamma_independence_cyclic5(pp):
    """acceptance.cpp:493-550: 70 converged for every gamma seed, same endpoint set within 1e-8"""
    sets = []
    for seed in (101, 102, 103):
        _, _, starts, h = homotopy(pp, read("cyclic5.sys"), "dd", seed=seed)
        sol = pp.track_all(h, starts)
        assert int(np.sum(sol.status == pp.SUCCESS)) == 70
        sets.append(sol.x_complex()[sol.status == pp.SUCCESS])
    for other in sets[1:]:
        used = np.zeros(len(other), bool)
        for x in sets[0]:
            d = np.max(np.abs(other - x), axis=1)
            d[used] = np.inf
            j = int(np.argmin(d))
            assert d[j] < 1e-8
            used[j] = True
