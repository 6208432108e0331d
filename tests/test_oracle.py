"""The C oracle (oracle/oracle.c) pinned against the reference: bit-exact against the golden
fixtures produced by the unmodified reference build (tests/golden/make_golden.py), and -- when the
reference build is present -- against the reference library directly on fresh random inputs."""

import numpy as np
import pytest

from conftest import golden, read

SQUARE_F = "1; x0^2 - 4;"
SQUARE_G = "1; x0^2 - 1;"
TRACK_KEYS = ["status", "reason", "steps", "newton_iters", "rejections", "x", "residual"]


def gamma_limbs(g: complex, prec: str):
    L = {"d": 1, "dd": 2, "qd": 4}[prec]
    a = np.zeros(2 * L)
    a[0], a[L] = g.real, g.imag
    return a


def need_ref(O):
    if O.ref is None:
        pytest.skip("reference build (oracle/_ref) not present")


@pytest.mark.parametrize("prec", ["d", "dd", "qd"])
@pytest.mark.parametrize("system", ["cyclic5", "cyclic10"])
def test_eval_matches_golden(oracle_mod, prec, system):
    O = oracle_mod
    g = golden(f"eval_{system}_{prec}")
    text = read(f"{system}.sys")
    need_ref(O)  # the oracle consumes the reference's plan tables
    plan = O.ref_plan(text, prec, g["gamma"])
    for i in range(g["points"].shape[0]):
        s, j = O.oracle_eval(plan, g["points"][i], g["t"][i])
        assert np.array_equal(s, g["sys"][i]), f"sys point {i}"
        assert np.array_equal(j, g["jac"][i]), f"jac point {i}"


@pytest.mark.parametrize("prec", ["d", "dd", "qd"])
@pytest.mark.parametrize("n", [1, 5, 10, 13])
def test_lsq_matches_golden(oracle_mod, prec, n):
    O = oracle_mod
    g = golden(f"lsq_n{n}_{prec}")
    for i in range(g["a"].shape[0]):
        x, ok = O.oracle_lsq(prec, g["a"][i], g["b"][i])
        assert ok == bool(g["ok"][i])
        assert np.array_equal(x, g["x"][i])
    assert not g["ok"].all()  # the fixture contains rank-deficient members


@pytest.mark.parametrize("prec", ["d", "dd", "qd"])
def test_arithmetic_bitwise_vs_reference(oracle_mod, prec):
    O = oracle_mod
    need_ref(O)
    rng = np.random.default_rng(7)
    L = O.LIMBS[prec]
    for _ in range(400):
        a, b = np.zeros(8), np.zeros(8)
        for arr in (a, b):
            for part in (0, L):
                arr[part] = rng.standard_normal() * 10.0 ** rng.integers(-6, 6)
                for l in range(1, L):
                    arr[part + l] = arr[part + l - 1] * rng.uniform(-1, 1) * 2.0 ** -53
        for op in range(11):
            aa = a.copy()
            if op == 5:
                aa[0] = abs(aa[0])
            assert np.array_equal(O.ref_arith(prec, op, aa, b), O.oracle_arith(prec, op, aa, b)), (op, aa, b)


def _track_golden(O, name, text, starts=None, g_text=None):
    g = golden(f"track_{name}")
    prec = str(g["prec"])
    gam = O.ref_random_gamma(int(g["gamma_seed"]))
    cfg = O.ref_defaults(prec)
    cfg.update(eval(str(g["cfg"])))
    plan = O.ref_plan(text, prec, gamma_limbs(gam, prec), g_text=g_text)
    lo, hi = int(g["lo"]), int(g["hi"])
    if starts is None:
        starts = np.stack([O.ref_td_solution(text, prec, i, plan["dim"]) for i in range(lo, hi)])
    r = O.oracle_track(plan, cfg, starts)
    for k in TRACK_KEYS:
        assert np.array_equal(r[k], g[k]), k
    return g


@pytest.mark.parametrize("name", ["cyclic5_d", "cyclic5_dd", "cyclic5_dd_seed101", "cyclic5_d_tight"])
def test_track_cyclic5_matches_golden(oracle_mod, name):
    O = oracle_mod
    need_ref(O)
    g = _track_golden(O, name, read("cyclic5.sys"))
    # the reference's acceptance facts (acceptance.cpp:493-550 and SURVEY.md 8c)
    if name != "cyclic5_d_tight":
        assert int(np.sum(g["status"] == 1)) == 70


def test_track_cyclic5_qd_subset(oracle_mod):
    O = oracle_mod
    need_ref(O)
    _track_golden(O, "cyclic5_qd", read("cyclic5.sys"))


def test_track_square_and_cyclic3(oracle_mod):
    O = oracle_mod
    need_ref(O)
    starts = np.array([[[1.0, 0.0]], [[-1.0, 0.0]]])
    g = _track_golden(O, "square_d", SQUARE_F, starts=starts, g_text=SQUARE_G)
    assert sorted(np.round(g["x"][:, 0, 0], 10).tolist()) == [-2.0, 2.0]
    _track_golden(O, "cyclic3_dd", O.ref_cyclic_text(3))


@pytest.mark.slow
def test_track_cyclic10_d_matches_golden(oracle_mod):
    O = oracle_mod
    need_ref(O)
    _track_golden(O, "cyclic10_d", read("cyclic10.sys"))


def test_reference_build_reproduces_golden(oracle_mod):
    """The fixtures are regenerable: the reference build gives the same bits today."""
    O = oracle_mod
    need_ref(O)
    g = golden("track_cyclic5_d")
    r = O.ref_track(read("cyclic5.sys"), "d", O.ref_random_gamma(1), lo=0, hi=120)
    for k in TRACK_KEYS:
        assert np.array_equal(r[k], g[k]), k
