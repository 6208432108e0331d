"""Host side of the product (no GPU needed): system grammar, decimal I/O, plan tables, start data,
gamma, TrackConfig -- each checked bit for bit against the reference build or its golden facts."""

import numpy as np
import pytest

from conftest import golden, read


def need_ref(O):
    if O.ref is None:
        pytest.skip("reference build (oracle/_ref) not present")


def test_random_gamma_matches_reference(pp, oracle_mod):
    need_ref(oracle_mod)
    for seed in (0, 1, 2, 3, 101, 102, 103, 12345, 2**63 + 5):
        assert pp.random_gamma(seed) == oracle_mod.ref_random_gamma(seed)
        assert abs(abs(pp.random_gamma(seed)) - 1.0) < 1e-15


@pytest.mark.parametrize("text", [
    "3; x0 + x1 + x2; x0*x1 - 2.5*x2^2; (1.5,-0.25)*x0*x1*x2 - 1;",
    "2\n# comment\nx0^3 + -x1;\n - 3 - x0*x0*x1 + 0.125e1 ;",
    "1; x0^2 - 4;",
    "2; x0*x1 + x1*x0 - 1; 3.14159265358979323846264338327950288419716939937510*x0^7 + x1;",
])
def test_parse_print_roundtrip_matches_reference(pp, oracle_mod, text):
    need_ref(oracle_mod)
    assert pp.parse_system(text).text() == oracle_mod.ref_print_system(text)


@pytest.mark.parametrize("bad", [
    "0; x0;", "2; x0 + x5;", "1; x0^0;", "1; x0 x0;", "1; 0*x0 + 1;", "1; x0 + 1", "", "1;", "1; x0^-2;",
    "1; (1,2*x0;",
])
def test_parse_errors_raise(pp, bad):
    with pytest.raises(pp.ParseError):
        pp.parse_system(bad)


def test_cyclic_generator(pp, oracle_mod):
    need_ref(oracle_mod)
    for n in (2, 3, 5, 8, 10):
        assert pp.cyclic_system(n).text() == oracle_mod.ref_cyclic_text(n)
    s = pp.cyclic_system(10).stats
    assert (s["dim"], s["n_polys"], s["n_monomials"], s["total_degree"]) == (10, 10, 92, 3628800)
    with pytest.raises(pp.InvalidArgument):
        pp.cyclic_system(1)


@pytest.mark.parametrize("prec", ["dd", "qd"])
def test_decimal_parse_and_print_match_reference(pp, oracle_mod, prec):
    need_ref(oracle_mod)
    rng = np.random.default_rng(3)
    samples = ["0", "1", "-0.5", "0.1", "1e-30", "6.02214076e23", "2.718281828459045235360287471352662497757247093699959574966967627",
               "123456789012345678901234567890.0987654321", "  7.25  "]
    samples += [f"{rng.uniform(-10, 10):.40f}" for _ in range(50)]
    for s in samples:
        a = oracle_mod.ref_parse_decimal(prec, s)
        b = pp.parse_decimal(prec, s)
        assert np.array_equal(a, b), s
        assert oracle_mod.ref_to_decimal(prec, a) == pp.to_decimal(prec, a)


@pytest.mark.parametrize("prec", ["d", "dd", "qd"])
@pytest.mark.parametrize("system", ["cyclic5.sys", "cyclic10.sys"])
def test_plan_matches_reference(pp, oracle_mod, prec, system):
    """build_plan (evaldiff.cpp:189-239): same term order, same coefficients bit for bit, same
    schedule counts (3k-5 position-product multiplications)."""
    need_ref(oracle_mod)
    text = read(system)
    f = pp.parse_system(text)
    g, _ = pp.total_degree_start(f, prec)
    gam = pp.random_gamma(1)
    h = pp.make_homotopy(f, g, gam, prec)
    ref = oracle_mod.ref_plan(text, prec, pp.gamma_limbs(gam, prec))
    assert np.array_equal(h.coefficients().reshape(-1), ref["coeff"].reshape(-1))
    info, rinfo = h.info, oracle_mod.ref_plan_info(text, prec)
    for k in ("dim", "n_polys", "n_terms", "mon_rows", "posprod_muls", "max_k", "jac_terms", "mon_steps"):
        assert info[k] == rinfo[k], k


def test_plan_geometry_table(pp):
    """SURVEY.md section 8 geometry: cyclic5/8/10 plan terms, mon rows, steps, cmul steps."""
    want = {5: (30, 89, 156, 83, 59), 8: (72, 311, 646, 456, 239), 10: (110, 579, 1283, 985, 469)}
    for n, (terms, rows, steps, cmul, jac) in want.items():
        f = pp.cyclic_system(n)
        g, _ = pp.total_degree_start(f, "d")
        info = pp.make_homotopy(f, g, pp.random_gamma(1), "d").info
        assert (info["n_terms"], info["mon_rows"], info["mon_steps"], info["cmul_steps"], info["jac_terms"]) == (
            terms, rows, steps, cmul, jac)


@pytest.mark.parametrize("prec", ["d", "dd", "qd"])
def test_total_degree_starts_match_reference(pp, oracle_mod, prec):
    need_ref(oracle_mod)
    text = read("cyclic10.sys")
    f = pp.parse_system(text)
    _, st = pp.total_degree_start(f, prec)
    assert st.count == 3628800
    for idx in (0, 1, 9, 10, 123456, 2000000, 3628799):
        assert np.array_equal(st.solution(idx), oracle_mod.ref_td_solution(text, prec, idx, 10))


@pytest.mark.parametrize("prec", ["d", "dd", "qd"])
def test_starts_from_root_tables(pp, prec):
    """pp_starts_roots (the reference StartData's own tables) enumerates exactly as
    total_degree_start: index -> tuple of roots, last variable fastest (homotopy.cpp:73-85)"""
    f = pp.parse_system(read("cyclic5.sys"))
    _, td = pp.total_degree_start(f, prec)
    deg = f.degrees
    roots = []
    for i, d in enumerate(deg):
        stride = int(np.prod(deg[i + 1:], dtype=np.int64))
        roots += [td.solution(r * stride)[i] for r in range(d)]
    st = pp.starts_from_roots(deg, np.array(roots), prec)
    assert st.count == td.count == 120
    for i in range(st.count):
        assert np.array_equal(st.solution(i), td.solution(i))
    with pytest.raises(pp.InvalidArgument):
        pp.starts_from_roots([1, 0], np.zeros((1, 2 * pp.LIMBS[prec])), prec)


def test_golden_start_pack_equals_total_degree(pp):
    """cyclic5_starts.txt (reference data) == total_degree_start<QD>(cyclic5) to ~1e-64."""
    f = pp.parse_system(read("cyclic5.sys"))
    _, st = pp.total_degree_start(f, "qd")
    rows = [ln for ln in read("cyclic5_starts.txt").splitlines() if ln.strip()]
    assert len(rows) == st.count == 120
    for i in (0, 1, 57, 119):
        vals = [float(v) for v in rows[i].replace("(", "").replace(")", "").split(",")]
        sol = st.solution(i)
        assert np.allclose(sol[:, 0], vals[0::2], atol=1e-15) and np.allclose(sol[:, 4], vals[1::2], atol=1e-15)


def test_make_homotopy_checks(pp):
    f = pp.parse_system("2; x0 + x1; x0*x1 - 1;")
    g, _ = pp.total_degree_start(f, "dd")
    with pytest.raises(pp.InvalidArgument):
        pp.make_homotopy(f, g, 1.5 + 0j, "dd")
    h3 = pp.parse_system("3; x0; x1; x2;")
    with pytest.raises(pp.InvalidArgument):
        pp.make_homotopy(f, h3, 1.0 + 0j, "dd")
    with pytest.raises(pp.InvalidArgument):
        pp.total_degree_start(pp.parse_system("2; x0 + x1;"), "d")  # not square


def test_track_config_defaults_and_validation(pp, oracle_mod):
    for prec in ("d", "dd", "qd"):
        c = pp.TrackConfig.defaults(prec)
        c.validate()
        if oracle_mod.ref is not None:
            r = oracle_mod.ref_defaults(prec)
            for k, v in r.items():
                assert getattr(c, k) == v, (prec, k)
    bad = [dict(h_min=0.2), dict(max_newton=0), dict(batch=0), dict(expand=0.5), dict(contract=1.0),
           dict(residual_tol=0.0), dict(h_max=0.2), dict(h_init=1e-9)]
    for kw in bad:
        c = pp.TrackConfig.defaults("d")
        for k, v in kw.items():
            setattr(c, k, v)
        with pytest.raises(pp.InvalidArgument):
            c.validate()


def test_solutions_jsonl_matches_the_reference_cli_format(pp, oracle_mod):
    """pp_solutions_jsonl writes the reference CLI's records (polypath_main.cpp:125-189): decimal
    coordinates that parse back bit for bit, to_decimal equal to the reference's, counts/summary"""
    import json

    g = golden("track_cyclic5_dd")
    n = len(g["status"])
    sol = pp.SolutionSet("dd", np.arange(n, dtype=np.uint64), g["status"], g["reason"], g["steps"],
                         g["newton_iters"], g["rejections"], g["x"], g["residual"], {"wall_ms": 12.5, "total_rounds": 7})
    lines = [json.loads(ln) for ln in sol.to_jsonl(pp.random_gamma(1), seed=1).splitlines()]
    recs, summ = lines[:-1], lines[-1]
    assert len(recs) == n and summ["type"] == "summary" and summ["paths"] == n
    assert summ["converged"] == 70 and summ["diverged"] == 50 and summ["failed"] == 0
    assert summ["precision"] == "dd" and summ["corrector_rounds"] == 7
    assert sorted(recs[0].keys()) == list(recs[0].keys())  # nlohmann's sorted key order
    for i, r in enumerate(recs):
        assert r["path"] == r["start"] == i and r["type"] == "solution"
        assert r["status"] == ("converged" if g["status"][i] == 1 else "diverged" if g["reason"][i] == 1 else "failed")
        assert r["annotation"] == pp.REASONS[g["reason"][i]]
        assert r["steps"] == g["steps"][i] and r["newton"] == g["newton_iters"][i]
        assert r["residual"] == float(g["residual"][i][0] + g["residual"][i][1])
        for v, (re, im) in enumerate(r["x"]):
            # 32 significant digits: the parsed value is within a couple of dd ulps of the limbs
            for txt, limbs in ((re, g["x"][i, v, :2]), (im, g["x"][i, v, 2:])):
                back = pp.parse_decimal("dd", txt)
                assert abs((back[0] - limbs[0]) + (back[1] - limbs[1])) <= 1e-30 * max(1.0, abs(limbs[0]))
    if oracle_mod.ref is not None:
        for i in (0, 3, 77):
            for v in range(5):
                assert recs[i]["x"][v][0] == oracle_mod.ref_to_decimal("dd", g["x"][i, v, :2])
                assert recs[i]["x"][v][1] == oracle_mod.ref_to_decimal("dd", g["x"][i, v, 2:])


@pytest.mark.parametrize("system", ["cyclic5", "cyclic10", "katsura12", "rand32"])
def test_warp_accumulation_lists(pp, system):
    """tail-mode tables (plan.cpp build_accumulation_lists): every contribution slot is summed by
    exactly one accumulator, each accumulator visits its slots in plan (term) order, H_p sums the
    terms of polynomial p, and dH_p/dx_v sums exactly the terms of p that contain x_v"""
    f = pp.parse_system(read(system + ".sys"))
    g, _ = pp.total_degree_start(f, "dd")
    h = pp.make_homotopy(f, g, pp.random_gamma(1), "dd")
    ts, off, idx = (pp.plan_table(h, k) for k in ("term_slot", "acc_off", "acc_idx"))
    ti = pp.plan_table(h, "term_info").reshape(-1, 4)
    pos = pp.plan_table(h, "pos")
    n, npoly, nt = f.dim, len(f.degrees), len(ti)
    assert len(ts) == nt + 1 and ts[-1] == len(idx) and len(off) == npoly + npoly * n + 1
    assert np.array_equal(np.sort(idx), np.arange(len(idx)))          # a partition of the slots
    for a in range(len(off) - 1):
        lst = idx[off[a]:off[a + 1]]
        assert np.all(np.diff(lst.astype(np.int64)) > 0)              # plan order
        if a < npoly:
            want = [ts[i] for i in range(nt) if ti[i, 0] == a]
        else:
            p, v = divmod(a - npoly, n)
            want = [ts[i] + 1 + j for i in range(nt) if ti[i, 0] == p
                    for j in range(ti[i, 1]) if (pos[ti[i, 2] + j] & 0xFFFF) == v]
        assert list(lst) == want


def test_compact_scan_known_answer(pp):
    """test_tracker.cpp:62-78 / acceptance.cpp:91-102: (0,1,0,-1,0) -> scan (1,1,2,2,3),
    job (1,2,3), path (0,2,4)"""
    r = pp.compact_scan([0, 1, 0, -1, 0])
    assert list(r["scan"]) == [1, 1, 2, 2, 3] and r["active_count"] == 3
    assert list(r["job_idx"]) == [1, 2, 3] and list(r["path_idx"]) == [0, 2, 4]
    assert pp.compact_scan([])["active_count"] == 0


def test_qd_add_network_matches_sequential_merge(tmp_path):
    """The quad-double addition's merge network (xprec.cuh qdi::add_i) against the step-by-step
    merge of the reference's algorithm (qdi::add_seq_i, xprec.hpp:325-382), bit for bit, on 2M
    random, structured and adversarial operand pairs (cancellation, ties, signed zeros, inf, NaN,
    unordered limbs).  The header is the same source the device code compiles."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "qd_add_check")
    subprocess.run(["g++", "-O2", "-std=c++20", "-ffp-contract=off",
                    "-I" + os.path.join(root, "paper_1505_00383_b200", "csrc"), "-o", exe,
                    os.path.join(root, "tests", "native", "qd_add_check.cpp")], check=True)
    out = subprocess.run([exe, "2000000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert " 0 mismatches" in out.stdout
