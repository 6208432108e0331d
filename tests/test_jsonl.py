"""Byte-exact JSON-lines records: pp_solutions_jsonl against the reference CLI's
writer -- record_json / emit_solutions of polypath_main.cpp:125-189 built with nlohmann::json 3.11
and the reference library's to_decimal (oracle/jsonl_ref.cpp -> oracle/_ref/libjsonref.so) -- on
the same records, line for line and byte for byte; and the number formatting on its own over a few
million doubles (nlohmann prints with Grisu2, which is not always the shortest representation)."""

import ctypes
import os
import struct

import numpy as np
import pytest

from conftest import ROOT, golden

LIB = os.path.join(ROOT, "oracle", "_ref", "libjsonref.so")


@pytest.fixture(scope="module")
def jref():
    if not os.path.exists(LIB):
        pytest.skip("oracle/_ref/libjsonref.so not built (needs the reference sources and a json.hpp)")
    lib = ctypes.CDLL(LIB)
    vp, sz = ctypes.c_void_p, ctypes.c_size_t
    lib.ref_json_doubles.argtypes = [vp, sz, ctypes.c_char_p, sz, ctypes.POINTER(sz)]
    lib.ref_solutions_jsonl.argtypes = [vp, ctypes.c_int, ctypes.c_uint32, vp, ctypes.c_uint64, ctypes.c_char_p,
                                        ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_char_p, sz,
                                        ctypes.POINTER(sz)]
    return lib


def _two_call(fn, *args):
    need = ctypes.c_size_t()
    fn(*args, None, 0, ctypes.byref(need))
    buf = ctypes.create_string_buffer(need.value)
    assert fn(*args, buf, need.value, ctypes.byref(need)) == 0
    return buf.value.decode()


def formatted(pp, jref, v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    ours = _two_call(pp.lib.pp_test_json_doubles, v.ctypes.data_as(ctypes.c_void_p), len(v))
    ref = _two_call(jref.ref_json_doubles, v.ctypes.data_as(ctypes.c_void_p), len(v))
    return ours.split("\n"), ref.split("\n")


def special_doubles():
    vals = [0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1e-4, 1e-5, 9.999e-5, 1.5e-5, 1e14, 1e15, 1e16, 123456789012345.0,
            1234567890123456.0, 3.2e9, 2.0 ** -1074, 2.0 ** -1022, 2.0 ** -1023, 1.7976931348623157e308, 2.0 ** 1023,
            5e-324, 1e308, 1e-308, 4.35, 0.3, 2.0 / 3.0, 100.0, 1e21, 1e22, 1e23, 9007199254740993.0,
            float("inf"), float("-inf"), float("nan")]
    vals += [10.0 ** k for k in range(-320, 309)] + [2.0 ** k for k in range(-1074, 1024)]
    vals += [float(f"{d}e{k}") for d in (1, 2, 5, 9.5, 1.25, 3.14159) for k in range(-20, 25)]
    return np.array(vals)


def test_number_format_matches_nlohmann(pp, jref):
    rng = np.random.default_rng(2026)
    sets = [special_doubles(),
            rng.integers(0, 2 ** 64 - 1, size=1_000_000, dtype=np.uint64).view(np.float64),  # any bit pattern
            rng.uniform(-1e3, 1e3, 300_000), rng.uniform(0, 1, 300_000) * 10.0 ** rng.integers(-20, 20, 300_000),
            np.round(rng.uniform(-1e6, 1e6, 100_000)),  # integral values
            np.exp(rng.uniform(-40, 40, 300_000))]
    for v in sets:
        ours, ref = formatted(pp, jref, v)
        bad = [i for i, (a, b) in enumerate(zip(ours, ref)) if a != b]
        assert len(ours) == len(ref)
        assert not bad, [(struct.pack("<d", v[i]).hex(), ours[i], ref[i]) for i in bad[:5]]


def golden_solution_set(pp, name):
    g = golden(name)
    prec = str(g["prec"])
    return pp.SolutionSet(prec, g["path_id"], g["status"], g["reason"], g["steps"], g["newton_iters"],
                          g["rejections"], g["x"], g["residual"], {"batches": 3, "total_rounds": 4242})


@pytest.mark.parametrize("name", ["track_cyclic5_d", "track_cyclic5_dd", "track_cyclic5_qd", "track_cyclic5_d_tight",
                                  "track_cyclic10_dd_far", "track_katsura12_d", "track_rand32_d", "track_cyclic8_d",
                                  "track_cyclic10_dd_prod"])
@pytest.mark.parametrize("wall_ms", [0.0, 1234.5678, 3.2e9, 1e-7])
def test_jsonl_lines_match_the_reference_cli(pp, jref, name, wall_ms):
    sol = golden_solution_set(pp, name)
    gamma = pp.random_gamma(1)
    ours = sol.to_jsonl(gamma, seed=7, command="solve", wall_ms=wall_ms)
    L = pp.LIMBS[sol.prec]
    gl = np.ascontiguousarray(pp.gamma_limbs(gamma, sol.prec))
    arrs = [np.ascontiguousarray(a) for a in (sol.path_id, sol.status, sol.reason, sol.steps, sol.newton_iters,
                                               sol.rejections, sol.x, sol.residual)]
    rec = pp.RecordsC(len(sol), len(sol), *[a.ctypes.data_as(ctypes.c_void_p) for a in arrs])
    ref = _two_call(jref.ref_solutions_jsonl, ctypes.cast(ctypes.pointer(rec), ctypes.c_void_p),
                    {"d": 0, "dd": 1, "qd": 2}[sol.prec], sol.x.shape[1], gl.ctypes.data_as(ctypes.c_void_p), 7,
                    b"solve", wall_ms, 3, 4242)
    assert L >= 1
    ol, rl = ours.splitlines(), ref.splitlines()
    assert len(ol) == len(rl) == len(sol) + 1
    for i, (a, b) in enumerate(zip(ol, rl)):
        assert a == b, (i, a[:300], b[:300])
    assert ours == ref


def test_jsonl_extreme_record_values(pp, jref):
    """failed paths with huge / tiny / non-finite residuals and large counters"""
    sol = golden_solution_set(pp, "track_cyclic5_d_tight")
    res = sol.residual.copy()
    res[:8, 0] = [1e300, 3.2e9, 1e-300, float("inf"), float("nan"), -0.0, 123456789.0, 2.0 ** -1074]
    sol.residual = res
    sol.steps = sol.steps.copy()
    sol.steps[0] = 2 ** 32 - 1
    test_sol = sol
    gamma = pp.random_gamma(3)
    ours = test_sol.to_jsonl(gamma, seed=2 ** 63, command="track", wall_ms=98765.4321)
    gl = np.ascontiguousarray(pp.gamma_limbs(gamma, "d"))
    arrs = [np.ascontiguousarray(a) for a in (sol.path_id, sol.status, sol.reason, sol.steps, sol.newton_iters,
                                               sol.rejections, sol.x, sol.residual)]
    rec = pp.RecordsC(len(sol), len(sol), *[a.ctypes.data_as(ctypes.c_void_p) for a in arrs])
    ref = _two_call(jref.ref_solutions_jsonl, ctypes.cast(ctypes.pointer(rec), ctypes.c_void_p), 0, sol.x.shape[1],
                    gl.ctypes.data_as(ctypes.c_void_p), 2 ** 63, b"track", 98765.4321, 3, 4242)
    assert ours == ref
