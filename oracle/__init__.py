"""TEST INFRASTRUCTURE ONLY -- the parity checker.

Two CPU implementations of the reference tracker, loaded by ctypes:

* ``ref``: the UNMODIFIED reference library (polypath) compiled from its own sources into
  ``oracle/_ref/libppref.so`` by ``oracle/Makefile`` (with ``oracle/ref_harness.cpp`` exposing its
  entry points), and
* ``orc``: ``oracle/liboracle.so``, the plain-C restatement in ``oracle/oracle.c``, pinned against
  ``ref`` and the golden fixtures in ``tests/golden``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference legs import this
package, and only as the checker or the timed CPU baseline.  The product never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libppref.so")
ORACLE_SO = os.path.join(HERE, "liboracle.so")
LIMBS = {"d": 1, "dd": 2, "qd": 4}
PREC = {"d": 0, "dd": 1, "qd": 2}

_vp, _u32, _u64, _i32, _dbl, _sz = (ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int,
                                    ctypes.c_double, ctypes.c_size_t)


def build(reference_root: str = "/root/reference/proj") -> None:
    """Compile liboracle.so and, when the reference sources are present, _ref/libppref.so."""
    targets = ["liboracle.so"]
    if os.path.isdir(reference_root):
        # the reference library, and its acceptance suite on the CPU tracker and through the
        # drop-in shim on libpp200.so (needs the CUDA library built first)
        targets += ["ref", "acceptance", "jsonref"]
    subprocess.run(["make", "-C", HERE, "-j8", f"REF={reference_root}", *targets], check=True,
                   stdout=subprocess.DEVNULL)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


class TrackConfigC(ctypes.Structure):
    _fields_ = [("residual_tol", _dbl), ("update_tol", _dbl), ("max_newton", ctypes.c_int32),
                ("expand_after", ctypes.c_int32), ("h_init", _dbl), ("h_min", _dbl), ("h_max", _dbl),
                ("expand", _dbl), ("contract", _dbl), ("divergence_bound", _dbl), ("max_steps", _u32),
                ("batch", _u32), ("workers", _u32), ("reserved", _u32)]


class RecordsC(ctypes.Structure):
    _fields_ = [("capacity", _u64), ("count", _u64)] + [(k, _vp) for k in
                                                         ("path_id", "status", "reason", "steps", "newton_iters",
                                                          "rejections", "x", "residual")]


class OraclePlanC(ctypes.Structure):
    _fields_ = [("L", _i32), ("dim", _i32), ("n_polys", _i32), ("n_terms", _i32), ("term_info", _vp),
                ("pos", _vp), ("coeff", _vp)]


class OracleCfgC(ctypes.Structure):
    _fields_ = [("residual_tol", _dbl), ("update_tol", _dbl), ("max_newton", _i32), ("expand_after", _i32),
                ("h_init", _dbl), ("h_min", _dbl), ("h_max", _dbl), ("expand", _dbl), ("contract", _dbl),
                ("divergence_bound", _dbl), ("max_steps", _u32)]


def _load(path):
    if not os.path.exists(path):
        return None
    return ctypes.CDLL(path)


ref = _load(REF_SO)
orc = _load(ORACLE_SO)

if ref is not None:
    ref.ref_last_error.restype = ctypes.c_char_p
    ref.ref_default_workers.restype = ctypes.c_uint
    ref.ref_track.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, _i32, _vp, ctypes.POINTER(TrackConfigC),
                              _u64, _u64, ctypes.POINTER(RecordsC), ctypes.POINTER(_dbl), ctypes.POINTER(_u64)]
    ref.ref_track_events.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, _i32, _vp,
                                     ctypes.POINTER(TrackConfigC), _u64, _u64, ctypes.POINTER(RecordsC), _vp, _u64,
                                     ctypes.POINTER(_u64)]
    ref.ref_newton.argtypes = [ctypes.c_char_p, ctypes.c_char_p, _i32, _vp, ctypes.POINTER(TrackConfigC), _u32, _vp, _vp,
                               _vp, _vp, ctypes.POINTER(_u32)]
    ref.ref_eval.argtypes = [ctypes.c_char_p, ctypes.c_char_p, _i32, _vp, _u32, _vp, _vp, _vp, _vp]
    ref.ref_lsq.argtypes = [_i32, _u32, _u32, _vp, _vp, _vp, _vp]
    ref.ref_td_solution.argtypes = [ctypes.c_char_p, _i32, _u64, _vp]
    ref.ref_arith.argtypes = [_i32, _i32, _vp, _vp, _vp]
    ref.ref_parse_decimal.argtypes = [_i32, ctypes.c_char_p, _vp]
    ref.ref_to_decimal.argtypes = [_i32, _vp, ctypes.c_char_p, _sz]
    ref.ref_plan_info.argtypes = [ctypes.c_char_p, ctypes.c_char_p, _i32, _vp, _vp]
    ref.ref_plan_terms.argtypes = [ctypes.c_char_p, ctypes.c_char_p, _i32, _vp, _vp, _vp, _vp, _vp]
    ref.ref_print_system.argtypes = [ctypes.c_char_p, ctypes.c_char_p, _sz]
    ref.ref_cyclic_text.argtypes = [_u32, ctypes.c_char_p, _sz]
    ref.ref_random_gamma.argtypes = [_u64, ctypes.POINTER(_dbl), ctypes.POINTER(_dbl)]
    ref.ref_track_config_defaults.argtypes = [_i32, ctypes.POINTER(TrackConfigC)]

if orc is not None:
    orc.oracle_eval.argtypes = [ctypes.POINTER(OraclePlanC), _vp, _vp, _vp, _vp]
    orc.oracle_lsq.argtypes = [_i32, _i32, _vp, _vp, _vp]
    orc.oracle_track_path.argtypes = [ctypes.POINTER(OraclePlanC), ctypes.POINTER(OracleCfgC), _vp, _vp, _vp, _vp]
    orc.oracle_arith.argtypes = [_i32, _i32, _vp, _vp, _vp]


def _need(lib, what):
    if lib is None:
        raise RuntimeError(f"{what} not built (run oracle.build())")
    return lib


def _chk(rc):
    if rc != 0:
        raise RuntimeError(f"reference harness error {rc}: {ref.ref_last_error().decode()}")


# ------------------------------------------------------------------------------------------------
# the reference build
# ------------------------------------------------------------------------------------------------
def ref_defaults(prec: str) -> dict:
    c = TrackConfigC()
    _need(ref, "reference build").ref_track_config_defaults(PREC[prec], ctypes.byref(c))
    return {k: getattr(c, k) for k, _ in TrackConfigC._fields_ if k != "reserved"}


def ref_random_gamma(seed: int) -> complex:
    re, im = _dbl(), _dbl()
    _need(ref, "reference build").ref_random_gamma(seed, ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


def ref_track(f_text: str, prec: str, gamma: complex, cfg: dict | None = None, lo: int = 0, hi: int | None = None,
              g_text: str | None = None, starts_text: str | None = None, workers: int = 1, batch: int = 64,
              count_hint: int | None = None):
    """track_all<R> of the reference on starts [lo, hi); returns dict of arrays (+ wall_ms)."""
    _need(ref, "reference build")
    c = TrackConfigC()
    ref.ref_track_config_defaults(PREC[prec], ctypes.byref(c))
    for k, v in (cfg or {}).items():
        setattr(c, k, v)
    c.workers = workers
    c.batch = batch
    L = LIMBS[prec]
    dim = int(f_text.strip().split(";")[0].split()[0]) if f_text.strip()[0].isdigit() else None
    hi_v = (1 << 64) - 1 if hi is None else hi
    cap = count_hint if count_hint is not None else (hi - lo if hi is not None else 1 << 16)
    arrs = dict(path_id=np.zeros(cap, np.uint64), status=np.zeros(cap, np.int8), reason=np.zeros(cap, np.uint8),
                steps=np.zeros(cap, np.uint32), newton_iters=np.zeros(cap, np.uint32),
                rejections=np.zeros(cap, np.uint32), x=np.zeros((cap, dim, 2 * L)), residual=np.zeros((cap, L)))
    rec = RecordsC(cap, 0, *[_ptr(arrs[k]) for k in ("path_id", "status", "reason", "steps", "newton_iters",
                                                      "rejections", "x", "residual")])
    g = np.array([gamma.real, gamma.imag])
    wall, rounds = _dbl(), _u64()
    _chk(ref.ref_track(f_text.encode(), g_text.encode() if g_text else None,
                       starts_text.encode() if starts_text else None, PREC[prec], _ptr(g), ctypes.byref(c), lo, hi_v,
                       ctypes.byref(rec), ctypes.byref(wall), ctypes.byref(rounds)))
    k = rec.count
    out = {key: v[:k].copy() for key, v in arrs.items()}
    out["wall_ms"] = wall.value
    out["total_rounds"] = rounds.value
    return out


EVENT_DTYPE = np.dtype([("path_id", np.uint64), ("t", np.float64), ("h", np.float64), ("newton_iters", np.uint32),
                        ("status", np.int8), ("accepted", np.uint8), ("reserved", np.uint8, 2)])


def ref_track_events(f_text: str, prec: str, gamma: complex, cfg: dict | None = None, lo: int = 0,
                     hi: int | None = None, batch: int = 64, ev_cap: int = 1 << 20):
    """track_all<R> of the reference with a ProgressSink collecting its StepEvents in emission order
    (tracker.cpp:312-315); returns (records dict, events as EVENT_DTYPE array)"""
    _need(ref, "reference build")
    c = TrackConfigC()
    ref.ref_track_config_defaults(PREC[prec], ctypes.byref(c))
    for k, v in (cfg or {}).items():
        setattr(c, k, v)
    c.workers = 1
    c.batch = batch
    L = LIMBS[prec]
    dim = int(f_text.strip().split(";")[0].split()[0])
    cap = hi - lo
    arrs = dict(path_id=np.zeros(cap, np.uint64), status=np.zeros(cap, np.int8), reason=np.zeros(cap, np.uint8),
                steps=np.zeros(cap, np.uint32), newton_iters=np.zeros(cap, np.uint32),
                rejections=np.zeros(cap, np.uint32), x=np.zeros((cap, dim, 2 * L)), residual=np.zeros((cap, L)))
    rec = RecordsC(cap, 0, *[_ptr(arrs[k]) for k in ("path_id", "status", "reason", "steps", "newton_iters",
                                                      "rejections", "x", "residual")])
    g = np.array([gamma.real, gamma.imag])
    ev = np.zeros(ev_cap, EVENT_DTYPE)
    n_ev = _u64()
    _chk(ref.ref_track_events(f_text.encode(), None, None, PREC[prec], _ptr(g), ctypes.byref(c), lo, hi,
                              ctypes.byref(rec), _ptr(ev), ev_cap, ctypes.byref(n_ev)))
    if n_ev.value > ev_cap:
        raise RuntimeError("event capacity exceeded")
    k = rec.count
    return {key: v[:k].copy() for key, v in arrs.items()}, ev[:n_ev.value].copy()


def ref_newton(f_text: str, prec: str, gamma_limbs: np.ndarray, t: np.ndarray, x: np.ndarray, cfg: dict | None = None,
               g_text: str | None = None):
    """PathBatch::set_prediction + newton_correct of the reference (tracker.hpp:135-136) for the
    pairs t [B][L], x [B][dim][2L]; returns (iterations, corrected, last iterates, rounds)"""
    _need(ref, "reference build")
    c = TrackConfigC()
    ref.ref_track_config_defaults(PREC[prec], ctypes.byref(c))
    for k, v in (cfg or {}).items():
        setattr(c, k, v)
    t = np.ascontiguousarray(t, dtype=np.float64)
    xo = np.ascontiguousarray(x, dtype=np.float64).copy()
    B = len(t)
    it = np.zeros(B, np.uint32)
    co = np.zeros(B, np.uint8)
    rounds = _u32()
    gl = np.ascontiguousarray(gamma_limbs, dtype=np.float64)
    _chk(ref.ref_newton(f_text.encode(), g_text.encode() if g_text else None, PREC[prec], _ptr(gl), ctypes.byref(c), B,
                        _ptr(t), _ptr(xo), _ptr(it), _ptr(co), ctypes.byref(rounds)))
    return it, co.astype(bool), xo, rounds.value


def ref_eval(f_text: str, prec: str, gamma_limbs: np.ndarray, points: np.ndarray, t: np.ndarray,
             g_text: str | None = None, n_polys: int | None = None):
    _need(ref, "reference build")
    B, dim = points.shape[0], points.shape[1]
    n_polys = n_polys or dim
    L = LIMBS[prec]
    sys = np.zeros((B, n_polys, 2 * L))
    jac = np.zeros((B, n_polys * dim, 2 * L))
    _chk(ref.ref_eval(f_text.encode(), g_text.encode() if g_text else None, PREC[prec],
                      _ptr(np.ascontiguousarray(gamma_limbs, dtype=np.float64)), B,
                      _ptr(np.ascontiguousarray(points)), _ptr(np.ascontiguousarray(t)), _ptr(sys), _ptr(jac)))
    return sys, jac


def ref_lsq(prec: str, a: np.ndarray, b: np.ndarray):
    _need(ref, "reference build")
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    B, n = a.shape[0], a.shape[1]
    x = np.zeros_like(b)
    ok = np.zeros(B, np.uint8)
    _chk(ref.ref_lsq(PREC[prec], n, B, _ptr(a), _ptr(b), _ptr(x), _ptr(ok)))
    return x, ok.astype(bool)


def ref_td_solution(f_text: str, prec: str, idx: int, dim: int) -> np.ndarray:
    out = np.zeros((dim, 2 * LIMBS[prec]))
    _chk(_need(ref, "reference build").ref_td_solution(f_text.encode(), PREC[prec], idx, _ptr(out)))
    return out


def ref_arith(prec: str, op: int, a, b) -> np.ndarray:
    out = np.zeros(8)
    _chk(_need(ref, "reference build").ref_arith(PREC[prec], op, _ptr(np.ascontiguousarray(a, dtype=np.float64)),
                                                 _ptr(np.ascontiguousarray(b, dtype=np.float64)), _ptr(out)))
    return out


def ref_parse_decimal(prec: str, s: str) -> np.ndarray:
    out = np.zeros(4)
    _chk(_need(ref, "reference build").ref_parse_decimal(PREC[prec], s.encode(), _ptr(out)))
    return out[: LIMBS[prec]]


def ref_to_decimal(prec: str, limbs) -> str:
    a = np.zeros(4)
    a[: len(limbs)] = limbs
    buf = ctypes.create_string_buffer(128)
    _chk(_need(ref, "reference build").ref_to_decimal(PREC[prec], _ptr(a), buf, 128))
    return buf.value.decode()


def ref_plan_info(f_text: str, prec: str, g_text: str | None = None):
    info = np.zeros(8, np.uint32)
    _chk(_need(ref, "reference build").ref_plan_info(f_text.encode(), g_text.encode() if g_text else None, PREC[prec],
                                                     _ptr(info), None))
    keys = ["dim", "n_polys", "n_terms", "mon_rows", "mon_steps", "posprod_muls", "jac_terms", "max_k"]
    return dict(zip(keys, (int(v) for v in info)))


def ref_plan(f_text: str, prec: str, gamma_limbs: np.ndarray, g_text: str | None = None) -> dict:
    """The reference build_plan as neutral SoA tables (the oracle's input)."""
    _need(ref, "reference build")
    counts = np.zeros(4, np.uint32)
    gl = np.ascontiguousarray(gamma_limbs, dtype=np.float64)
    gt = g_text.encode() if g_text else None
    _chk(ref.ref_plan_terms(f_text.encode(), gt, PREC[prec], _ptr(gl), None, None, None, _ptr(counts)))
    dim, n_polys, n_terms, n_pos = (int(v) for v in counts)
    L = LIMBS[prec]
    ti = np.zeros(4 * max(n_terms, 1), np.int32)
    pos = np.zeros(max(n_pos, 1), np.uint32)
    coeff = np.zeros((max(n_terms, 1), 2, 2 * L))
    _chk(ref.ref_plan_terms(f_text.encode(), gt, PREC[prec], _ptr(gl), _ptr(ti), _ptr(pos), _ptr(coeff),
                            _ptr(counts)))
    return dict(L=L, dim=dim, n_polys=n_polys, n_terms=n_terms, term_info=ti, pos=pos, coeff=coeff)


def ref_print_system(text: str) -> str:
    buf = ctypes.create_string_buffer(1 << 20)
    _chk(_need(ref, "reference build").ref_print_system(text.encode(), buf, 1 << 20))
    return buf.value.decode()


def ref_cyclic_text(n: int) -> str:
    buf = ctypes.create_string_buffer(1 << 20)
    _chk(_need(ref, "reference build").ref_cyclic_text(n, buf, 1 << 20))
    return buf.value.decode()


# ------------------------------------------------------------------------------------------------
# the C restatement
# ------------------------------------------------------------------------------------------------
def _plan_c(plan: dict):
    keep = (plan["term_info"], plan["pos"], np.ascontiguousarray(plan["coeff"]))
    c = OraclePlanC(plan["L"], plan["dim"], plan["n_polys"], plan["n_terms"], _ptr(keep[0]), _ptr(keep[1]),
                    _ptr(keep[2]))
    return c, keep


def oracle_eval(plan: dict, x: np.ndarray, t: np.ndarray):
    _need(orc, "oracle")
    pc, keep = _plan_c(plan)
    L = plan["L"]
    sys = np.zeros((plan["n_polys"], 2 * L))
    jac = np.zeros((plan["n_polys"] * plan["dim"], 2 * L))
    orc.oracle_eval(ctypes.byref(pc), _ptr(np.ascontiguousarray(x)), _ptr(np.ascontiguousarray(t)), _ptr(sys),
                    _ptr(jac))
    return sys, jac


def oracle_lsq(prec: str, a: np.ndarray, b: np.ndarray):
    _need(orc, "oracle")
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    ok = orc.oracle_lsq(LIMBS[prec], a.shape[0], _ptr(a), _ptr(b), _ptr(x))
    return x, bool(ok)


def oracle_arith(prec: str, op: int, a, b) -> np.ndarray:
    out = np.zeros(8)
    _need(orc, "oracle").oracle_arith(LIMBS[prec], op, _ptr(np.ascontiguousarray(a, dtype=np.float64)),
                                      _ptr(np.ascontiguousarray(b, dtype=np.float64)), _ptr(out))
    return out


def oracle_track(plan: dict, cfg: dict, starts: np.ndarray):
    """One record per start row ([count][dim][2L] limbs), tracked independently."""
    _need(orc, "oracle")
    pc, keep = _plan_c(plan)
    oc = OracleCfgC(*[cfg[k] for k, _ in OracleCfgC._fields_])
    count, dim = starts.shape[0], plan["dim"]
    L = plan["L"]
    x = np.zeros((count, dim, 2 * L))
    res = np.zeros((count, L))
    info = np.zeros((count, 5), np.int32)
    for i in range(count):
        s = np.ascontiguousarray(starts[i])
        orc.oracle_track_path(ctypes.byref(pc), ctypes.byref(oc), _ptr(s), _ptr(x[i]), _ptr(res[i]), _ptr(info[i]))
    return dict(status=info[:, 0].astype(np.int8), reason=info[:, 1].astype(np.uint8),
                steps=info[:, 2].astype(np.uint32), newton_iters=info[:, 3].astype(np.uint32),
                rejections=info[:, 4].astype(np.uint32), x=x, residual=res)
