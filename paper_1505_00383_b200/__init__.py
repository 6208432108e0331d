"""B200-native many-path polynomial-homotopy tracker.

Python mirror of the reference's drop-in API for the `track_all` hot path
(reference: proj/include/polypath/{polysys,homotopy,tracker}.hpp), over the C ABI of
``libpp200.so`` (include/pp200.h).  All numerics run in the CUDA library; this module only
marshals buffers.  There is no CPU fallback: without the built library the import fails, and
without a CUDA device the tracking calls raise ``CudaError``.

    f = parse_system(open("cyclic10.sys").read())
    g, starts = total_degree_start(f, "dd")
    h = make_homotopy(f, g, random_gamma(1), "dd")
    sol = track_all(h, starts, TrackConfig.defaults("dd"))
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field, fields

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PP200_LIB") or os.path.join(_HERE, "libpp200.so")

PRECISIONS = {"d": 0, "dd": 1, "qd": 2}
LIMBS = {"d": 1, "dd": 2, "qd": 4}

# PathStatus / FailReason (tracker.hpp:16-25)
FAILED, ACTIVE, SUCCESS = -1, 0, 1
REASONS = ["converged", "diverged", "step-underflow", "max-steps", "singular", "no-certificate"]


class PPError(RuntimeError):
    code = -99


class InvalidArgument(PPError, ValueError):
    """std::invalid_argument in the reference."""

    code = -1


class ParseError(PPError):
    """polypath::ParseError in the reference."""

    code = -2


class CudaError(PPError):
    code = -3


_ERRORS = {-1: InvalidArgument, -2: ParseError, -3: CudaError}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first (python -c 'import __graft_entry__ as g; g.build()')"
        )
    return ctypes.CDLL(LIB_PATH)


lib = _load()


class TrackConfigC(ctypes.Structure):
    _fields_ = [
        ("residual_tol", ctypes.c_double),
        ("update_tol", ctypes.c_double),
        ("max_newton", ctypes.c_int32),
        ("expand_after", ctypes.c_int32),
        ("h_init", ctypes.c_double),
        ("h_min", ctypes.c_double),
        ("h_max", ctypes.c_double),
        ("expand", ctypes.c_double),
        ("contract", ctypes.c_double),
        ("divergence_bound", ctypes.c_double),
        ("max_steps", ctypes.c_uint32),
        ("batch", ctypes.c_uint32),
        ("workers", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
    ]


class RecordsC(ctypes.Structure):
    _fields_ = [
        ("capacity", ctypes.c_uint64),
        ("count", ctypes.c_uint64),
        ("path_id", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
        ("reason", ctypes.c_void_p),
        ("steps", ctypes.c_void_p),
        ("newton_iters", ctypes.c_void_p),
        ("rejections", ctypes.c_void_p),
        ("x", ctypes.c_void_p),
        ("residual", ctypes.c_void_p),
    ]


class RunStatsC(ctypes.Structure):
    _fields_ = [
        ("paths", ctypes.c_uint64),
        ("batches", ctypes.c_uint64),
        ("total_rounds", ctypes.c_uint64),
        ("newton_iters", ctypes.c_uint64),
        ("device_ms", ctypes.c_double),
        ("h2d_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("wall_ms", ctypes.c_double),
        ("h2d_bytes", ctypes.c_uint64),
        ("d2h_bytes", ctypes.c_uint64),
        ("slots", ctypes.c_uint32),
        ("kernel_launches", ctypes.c_uint32),
        ("evals", ctypes.c_uint64),
        ("solves", ctypes.c_uint64),
        ("eval_ms", ctypes.c_double),
        ("lsq_ms", ctypes.c_double),
        ("step_ms", ctypes.c_double),
        ("events", ctypes.c_uint64),
    ]


class ShardC(ctypes.Structure):
    _fields_ = [("index", ctypes.c_uint32), ("count", ctypes.c_uint32), ("block", ctypes.c_uint64)]


class StepEventC(ctypes.Structure):
    """StepEvent (tracker.hpp:62-69), pp_step_event"""
    _fields_ = [("path_id", ctypes.c_uint64), ("t", ctypes.c_double), ("h", ctypes.c_double),
                ("newton_iters", ctypes.c_uint32), ("status", ctypes.c_int8), ("accepted", ctypes.c_uint8),
                ("reserved", ctypes.c_uint8 * 2)]


EVENT_DTYPE = np.dtype([("path_id", np.uint64), ("t", np.float64), ("h", np.float64), ("newton_iters", np.uint32),
                        ("status", np.int8), ("accepted", np.uint8), ("reserved", np.uint8, 2)])
assert EVENT_DTYPE.itemsize == ctypes.sizeof(StepEventC) == 32
EventSinkFn = ctypes.CFUNCTYPE(None, ctypes.POINTER(StepEventC), ctypes.c_uint64, ctypes.c_void_p)


_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_u32, _u64, _i32, _dbl = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
_P = ctypes.POINTER


def _sig(name, res, *args):
    fn = getattr(lib, name)
    fn.restype = res
    fn.argtypes = list(args)
    return fn


_sig("pp_version", ctypes.c_char_p)
_sig("pp_last_error", ctypes.c_char_p)
_sig("pp_limbs", _i32, _i32)
_sig("pp_system_parse", _i32, ctypes.c_char_p, _sz, _P(_vp))
_sig("pp_system_cyclic", _i32, _u32, _P(_vp))
_sig("pp_system_from_terms", _i32, _u32, _u32, _vp, _vp, _vp, _vp, _P(_vp))
_sig("pp_device_count", _i32)
_sig("pp_device_init", _i32, _i32)
_sig("pp_test_json_doubles", _i32, _vp, _sz, ctypes.c_char_p, _sz, _P(_sz))
_sig("pp_test_newton", _i32, _vp, _P(TrackConfigC), _u32, _vp, _vp, _vp, _vp, _vp, _i32)
_sig("pp_system_print", _i32, _vp, ctypes.c_char_p, _sz, _P(_sz))
_sig("pp_system_stats", _i32, _vp, _P(_u32), _P(_u32), _P(_u64), _P(_u64), _P(_i32))
_sig("pp_system_degrees", _i32, _vp, _vp)
_sig("pp_system_free", None, _vp)
_sig("pp_random_gamma", None, _u64, _P(_dbl), _P(_dbl))
_sig("pp_total_degree_start", _i32, _vp, _i32, _P(_vp), _P(_vp))
_sig("pp_load_start_data", _i32, _vp, _i32, ctypes.c_char_p, _sz, _dbl, _i32, _P(_vp), _vp, _vp, _u64, _P(_u64))
_sig("pp_starts_explicit", _i32, _i32, _u32, _u64, _vp, _P(_vp))
_sig("pp_starts_roots", _i32, _i32, _u32, _vp, _vp, _P(_vp))
_sig("pp_starts_count", _u64, _vp)
_sig("pp_starts_solution", _i32, _vp, _u64, _vp)
_sig("pp_starts_free", None, _vp)
_sig("pp_make_homotopy", _i32, _vp, _vp, _i32, _vp, _P(_vp))
_sig("pp_homotopy_info", _i32, _vp, _P(_u32), _P(_u32), _P(_u32), _P(_u32), _P(_u32), _P(_u64))
_sig("pp_homotopy_counts", _i32, _vp, _vp)
_sig("pp_homotopy_free", None, _vp)
_sig("pp_track_config_defaults", None, _i32, _P(TrackConfigC))
_sig("pp_track_config_validate", _i32, _P(TrackConfigC))
_sig("pp_track_all", _i32, _vp, _vp, _P(TrackConfigC), _u64, _u64, _i32, _P(RecordsC), _P(RunStatsC))
_sig("pp_track_all_ex", _i32, _vp, _vp, _P(TrackConfigC), _u64, _u64, _P(ShardC), EventSinkFn, _vp, _i32, _P(RecordsC),
     _P(RunStatsC))
_sig("pp_shard_size", _u64, _u64, _u64, _P(ShardC))
_sig("pp_solutions_jsonl", _i32, _vp, _i32, _u32, _vp, _u64, ctypes.c_char_p, _dbl, _u64, _u64, ctypes.c_char_p,
     _sz, _P(_sz))
_sig("pp_to_decimal", _i32, _i32, _vp, ctypes.c_char_p, _sz)
_sig("pp_bench_eval", _i32, _vp, _u64, _u32, _u32, _i32, _P(_dbl), _P(_u64))
_sig("pp_eval_batch", _i32, _vp, _u32, _vp, _vp, _vp, _vp, _i32)
_sig("pp_lsq_batch", _i32, _i32, _u32, _u32, _vp, _vp, _vp, _vp, _i32)
_sig("pp_lsq_batch_mn", _i32, _i32, _u32, _u32, _u32, _vp, _vp, _vp, _vp, _vp, _vp, _i32)
_sig("pp_test_arith", _i32, _i32, _i32, _vp, _vp, _vp)
_sig("pp_test_parse_decimal", _i32, _i32, ctypes.c_char_p, _vp)
_sig("pp_test_to_decimal", _i32, _i32, _vp, ctypes.c_char_p, _sz)
_sig("pp_test_plan_coeffs", _i32, _vp, _vp, _sz)
_sig("pp_test_plan_tables", _i32, _vp, _i32, _vp, _sz, _P(_sz))
_sig("pp_fp64_peak", _i32, _i32, _P(_dbl))

EXPORTED = [
    "pp_version", "pp_last_error", "pp_limbs", "pp_system_parse", "pp_system_cyclic", "pp_system_print",
    "pp_system_stats", "pp_system_degrees", "pp_system_free", "pp_random_gamma", "pp_total_degree_start",
    "pp_load_start_data", "pp_starts_explicit", "pp_starts_roots", "pp_starts_count", "pp_starts_solution", "pp_starts_free",
    "pp_make_homotopy", "pp_homotopy_info", "pp_homotopy_free", "pp_track_config_defaults",
    "pp_track_config_validate", "pp_track_all", "pp_eval_batch", "pp_lsq_batch", "pp_solutions_jsonl",
    "pp_to_decimal", "pp_bench_eval", "pp_track_all_ex", "pp_shard_size", "pp_system_from_terms", "pp_device_count", "pp_lsq_batch_mn", "pp_device_init",
]


def _check(rc):
    if rc != 0:
        msg = lib.pp_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, PPError)(f"pp200 error {rc}: {msg}")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


def _prec(p) -> int:
    if isinstance(p, int):
        return p
    return PRECISIONS[p]


def _pname(p) -> str:
    return {0: "d", 1: "dd", 2: "qd"}[_prec(p)]


class System:
    """PolySystem (polysys.hpp:41-51): owned handle to a parsed system."""

    def __init__(self, handle):
        self._h = _vp(handle)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.pp_system_free(self._h)
            self._h = None

    @property
    def stats(self):
        d, np_, = _u32(), _u32()
        nm, td, of = _u64(), _u64(), _i32()
        _check(lib.pp_system_stats(self._h, ctypes.byref(d), ctypes.byref(np_), ctypes.byref(nm), ctypes.byref(td),
                                   ctypes.byref(of)))
        return {"dim": d.value, "n_polys": np_.value, "n_monomials": nm.value, "total_degree": td.value,
                "total_degree_overflow": bool(of.value)}

    @property
    def dim(self) -> int:
        return self.stats["dim"]

    @property
    def degrees(self):
        out = np.zeros(self.stats["n_polys"], dtype=np.uint32)
        _check(lib.pp_system_degrees(self._h, _ptr(out)))
        return out.tolist()

    def text(self) -> str:
        need = _sz()
        lib.pp_system_print(self._h, None, 0, ctypes.byref(need))
        buf = ctypes.create_string_buffer(need.value)
        _check(lib.pp_system_print(self._h, buf, need.value, ctypes.byref(need)))
        return buf.value.decode()


def parse_system(text: str) -> System:
    """parse_system (polysys.cpp:117-252); raises ParseError with line/column."""
    raw = text.encode()
    h = _vp()
    _check(lib.pp_system_parse(raw, len(raw), ctypes.byref(h)))
    return System(h.value)


def cyclic_system(n: int) -> System:
    """cyclic_system (polysys.cpp:315-336)."""
    h = _vp()
    _check(lib.pp_system_cyclic(n, ctypes.byref(h)))
    return System(h.value)


def system_from_terms(dim: int, polys) -> System:
    """PolySystem from terms without a text round trip (pp_system_from_terms): polys is a list of
    polynomials, each a list of (coeff, [(var, exp), ...]) with coeff a complex or 8 QD limbs
    (re limbs, im limbs)."""
    counts, nf, fac, co = [], [], [], []
    for poly in polys:
        counts.append(len(poly))
        for c, mono in poly:
            limbs = np.zeros(8)
            if np.isscalar(c):
                limbs[0], limbs[4] = complex(c).real, complex(c).imag
            else:
                limbs[:] = np.asarray(c, dtype=np.float64)
            co.append(limbs)
            nf.append(len(mono))
            for v, e in mono:
                fac += [v, e]
    arrs = [np.asarray(counts, np.uint32), np.asarray(nf, np.uint32), np.asarray(fac or [0], np.uint32),
            np.asarray(co if co else np.zeros((1, 8)), np.float64)]
    out = _vp()
    _check(lib.pp_system_from_terms(dim, len(polys), *[_ptr(a) for a in arrs], ctypes.byref(out)))
    return System(out.value)


def device_count() -> int:
    return int(lib.pp_device_count())


def device_init(device: int = 0) -> None:
    """create the device context and load the kernels ahead of the first track_all (pp_device_init)"""
    _check(lib.pp_device_init(device))


def random_gamma(seed: int) -> complex:
    """random_gamma (homotopy.cpp:34-40)."""
    re, im = _dbl(), _dbl()
    lib.pp_random_gamma(seed, ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


class Starts:
    """StartData<R> (homotopy.hpp:38-49)."""

    def __init__(self, handle, prec, dim):
        self._h = _vp(handle)
        self.prec = _pname(prec)
        self.dim = dim

    def __del__(self):
        if getattr(self, "_h", None):
            lib.pp_starts_free(self._h)
            self._h = None

    @property
    def count(self) -> int:
        return lib.pp_starts_count(self._h)

    def __len__(self):
        return self.count

    def solution(self, index: int) -> np.ndarray:
        """StartData::solution (homotopy.cpp:73-85), limbs [dim][2L]."""
        out = np.zeros((self.dim, 2 * LIMBS[self.prec]))
        _check(lib.pp_starts_solution(self._h, index, _ptr(out)))
        return out


def total_degree_start(f: System, prec="dd"):
    """total_degree_start<R> (homotopy.cpp:87-113) -> (g, starts)."""
    g, s = _vp(), _vp()
    _check(lib.pp_total_degree_start(f._h, _prec(prec), ctypes.byref(g), ctypes.byref(s)))
    return System(g.value), Starts(s.value, prec, f.dim)


def explicit_starts(x: np.ndarray, prec="dd") -> Starts:
    """Explicit start list (StartProvenance::file): x is [count][dim][2L] limbs."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    count, dim = x.shape[0], x.shape[1]
    s = _vp()
    _check(lib.pp_starts_explicit(_prec(prec), dim, count, _ptr(x), ctypes.byref(s)))
    return Starts(s.value, prec, dim)


def starts_from_roots(degrees, roots: np.ndarray, prec="dd") -> Starts:
    """StartData<R> in total-degree mode from its own tables (homotopy.hpp:38-49): degrees[dim]
    and the per-variable root tables concatenated as [sum(degrees)][2L] limbs."""
    deg = np.ascontiguousarray(degrees, dtype=np.uint32)
    r = np.ascontiguousarray(roots, dtype=np.float64)
    if r.shape[0] != int(deg.sum()):
        raise InvalidArgument("starts_from_roots: root tables do not match the degrees")
    s = _vp()
    _check(lib.pp_starts_roots(_prec(prec), len(deg), _ptr(deg), _ptr(r), ctypes.byref(s)))
    return Starts(s.value, prec, len(deg))


def load_start_data(g: System, text: str, prec="dd", start_tol=1e-8, device=0):
    """load_start_data<R>(g, parse_solutions(text)) (homotopy.cpp:115-140); returns
    (starts, [(index, residual) of rejected candidates])."""
    raw = text.encode()
    cap = max(1, raw.count(b"\n") + 1)
    idx = np.zeros(cap, dtype=np.uint64)
    res = np.zeros(cap)
    nrej = _u64()
    s = _vp()
    _check(lib.pp_load_start_data(g._h, _prec(prec), raw, len(raw), start_tol, device, ctypes.byref(s), _ptr(idx),
                                  _ptr(res), cap, ctypes.byref(nrej)))
    k = min(nrej.value, cap)
    return Starts(s.value, prec, g.dim), [(int(idx[i]), float(res[i])) for i in range(k)]


def gamma_limbs(gamma: complex, prec) -> np.ndarray:
    """A double-valued gamma widened to the level (exact), as 2L limbs."""
    L = LIMBS[_pname(prec)]
    g = np.zeros(2 * L)
    g[0], g[L] = gamma.real, gamma.imag
    return g


class Homotopy:
    """HomotopyInstance<R> (homotopy.hpp:16-22) with its device-resident plan."""

    def __init__(self, handle, prec, f, g):
        self._h = _vp(handle)
        self.prec = _pname(prec)
        self.f, self.g = f, g

    def __del__(self):
        if getattr(self, "_h", None):
            lib.pp_homotopy_free(self._h)
            self._h = None

    @property
    def info(self):
        v = [_u32() for _ in range(5)]
        pm = _u64()
        _check(lib.pp_homotopy_info(self._h, *[ctypes.byref(x) for x in v], ctypes.byref(pm)))
        keys = ["dim", "n_polys", "n_terms", "mon_rows", "max_k"]
        out = {k: x.value for k, x in zip(keys, v)}
        out["posprod_muls"] = pm.value
        c = np.zeros(5, dtype=np.uint64)
        _check(lib.pp_homotopy_counts(self._h, _ptr(c)))
        out.update(mon_steps=int(c[0]), cmul_steps=int(c[1]), jac_terms=int(c[2]), jac_scaled=int(c[3]),
                   n_base=int(c[4]))
        return out

    def coefficients(self) -> np.ndarray:
        """per term (c_start, c_target) limbs, [terms][2][2L]"""
        L = LIMBS[self.prec]
        n = self.info["n_terms"]
        out = np.zeros((n, 2, 2 * L))
        _check(lib.pp_test_plan_coeffs(self._h, _ptr(out), out.size))
        return out


def plan_table(h: "Homotopy", which: str) -> np.ndarray:
    """test hook: a plan table (term_slot, acc_off, acc_idx, pos, term_info) as an array"""
    code = {"term_slot": 0, "acc_off": 1, "acc_idx": 2, "pos": 3, "term_info": 4}[which]
    cnt = _sz()
    lib.pp_test_plan_tables(h._h, code, None, 0, ctypes.byref(cnt))
    out = np.zeros(max(1, cnt.value), dtype=np.uint32)
    _check(lib.pp_test_plan_tables(h._h, code, _ptr(out), out.size, ctypes.byref(cnt)))
    return out[: cnt.value]


def make_homotopy(f: System, g: System, gamma, prec="dd") -> Homotopy:
    """make_homotopy<R>(f, g, gamma) (homotopy.cpp:7-20); gamma is a complex (widened exactly)
    or a 2L limb array."""
    gl = gamma if isinstance(gamma, np.ndarray) else gamma_limbs(complex(gamma), prec)
    gl = np.ascontiguousarray(gl, dtype=np.float64)
    h = _vp()
    _check(lib.pp_make_homotopy(f._h, g._h, _prec(prec), _ptr(gl), ctypes.byref(h)))
    return Homotopy(h.value, prec, f, g)


@dataclass
class TrackConfig:
    """TrackConfig (tracker.hpp:29-46)."""

    residual_tol: float = 1e-8
    update_tol: float = 1e-8
    max_newton: int = 3
    expand_after: int = 2
    h_init: float = 0.05
    h_min: float = 1e-6
    h_max: float = 0.1
    expand: float = 1.5
    contract: float = 0.5
    divergence_bound: float = 1e8
    max_steps: int = 10000
    batch: int = 64
    workers: int = 1

    @staticmethod
    def defaults(prec) -> "TrackConfig":
        c = TrackConfigC()
        lib.pp_track_config_defaults(_prec(prec), ctypes.byref(c))
        return TrackConfig(**{f.name: getattr(c, f.name) for f in fields(TrackConfig)})

    def to_c(self) -> TrackConfigC:
        c = TrackConfigC()
        for f in fields(self):
            setattr(c, f.name, getattr(self, f.name))
        return c

    def validate(self):
        c = self.to_c()
        _check(lib.pp_track_config_validate(ctypes.byref(c)))


@dataclass
class SolutionSet:
    """SolutionSet<R> (tracker.hpp:89-94) as arrays; record i is start lo+i."""

    prec: str
    path_id: np.ndarray
    status: np.ndarray
    reason: np.ndarray
    steps: np.ndarray
    newton_iters: np.ndarray
    rejections: np.ndarray
    x: np.ndarray  # [count][dim][2L]
    residual: np.ndarray  # [count][L]
    stats: dict = field(default_factory=dict)

    def __len__(self):
        return len(self.path_id)

    def x_complex(self) -> np.ndarray:
        """endpoints rounded to complex128 (to_double of each component)"""
        L = LIMBS[self.prec]
        re = self.x[:, :, :L]
        im = self.x[:, :, L:]
        if L == 1:
            return re[..., 0] + 1j * im[..., 0]
        if L == 2:
            return (re[..., 0] + re[..., 1]) + 1j * (im[..., 0] + im[..., 1])
        return (((re[..., 3] + re[..., 2]) + re[..., 1]) + re[..., 0]) + 1j * (
            ((im[..., 3] + im[..., 2]) + im[..., 1]) + im[..., 0])

    def to_jsonl(self, gamma, seed: int = 1, command: str = "solve", wall_ms: float | None = None) -> str:
        """The reference CLI's output (polypath_main.cpp:125-189): one JSON "solution" line per
        record with full-precision decimal coordinates, then the "summary" line.  gamma is the
        homotopy's gamma (complex, or 2L limbs)."""
        L = LIMBS[self.prec]
        g = np.ascontiguousarray(gamma_limbs(gamma, self.prec) if np.isscalar(gamma) else gamma, dtype=np.float64)
        arrs = [np.ascontiguousarray(a) for a in (self.path_id, self.status, self.reason, self.steps,
                                                   self.newton_iters, self.rejections, self.x, self.residual)]
        rec = RecordsC(len(self), len(self), *[_ptr(a) for a in arrs])
        dim = self.x.shape[1] if self.x.ndim == 3 else 0
        wall = self.stats.get("wall_ms", 0.0) if wall_ms is None else wall_ms
        args = (ctypes.byref(rec), _prec(self.prec), dim, _ptr(g), seed, command.encode(), float(wall),
                int(self.stats.get("batches", 1)), int(self.stats.get("total_rounds", 0)))
        need = _sz()
        rc = lib.pp_solutions_jsonl(*args, None, 0, ctypes.byref(need))
        if rc not in (0, -5):
            _check(rc)
        buf = ctypes.create_string_buffer(need.value)
        _check(lib.pp_solutions_jsonl(*args, buf, need.value, ctypes.byref(need)))
        del L
        return buf.value.decode()

    def counts(self):
        out = {"converged": int(np.sum(self.status == SUCCESS))}
        for r, name in enumerate(REASONS[1:], start=1):
            out[name] = int(np.sum((self.status == FAILED) & (self.reason == r)))
        return out


class Records:
    """Preallocated host record buffers (optionally pinned by the caller)."""

    def __init__(self, capacity: int, dim: int, prec):
        L = LIMBS[_pname(prec)]
        self.prec = _pname(prec)
        self.path_id = np.zeros(capacity, dtype=np.uint64)
        self.status = np.zeros(capacity, dtype=np.int8)
        self.reason = np.zeros(capacity, dtype=np.uint8)
        self.steps = np.zeros(capacity, dtype=np.uint32)
        self.newton_iters = np.zeros(capacity, dtype=np.uint32)
        self.rejections = np.zeros(capacity, dtype=np.uint32)
        self.x = np.zeros((capacity, dim, 2 * L))
        self.residual = np.zeros((capacity, L))
        self.c = RecordsC(capacity, 0, _ptr(self.path_id), _ptr(self.status), _ptr(self.reason), _ptr(self.steps),
                          _ptr(self.newton_iters), _ptr(self.rejections), _ptr(self.x), _ptr(self.residual))

    def solution_set(self, stats: dict) -> SolutionSet:
        k = self.c.count
        return SolutionSet(self.prec, self.path_id[:k].copy(), self.status[:k].copy(), self.reason[:k].copy(),
                           self.steps[:k].copy(), self.newton_iters[:k].copy(), self.rejections[:k].copy(),
                           self.x[:k].copy(), self.residual[:k].copy(), stats)


def shard_size(lo: int, hi: int, shard: tuple[int, int, int] | None) -> int:
    """number of start indices of [lo, hi) in the block-cyclic shard (index, count, block)"""
    sh = ShardC(*shard) if shard is not None else None
    return int(lib.pp_shard_size(lo, hi, ctypes.byref(sh) if sh is not None else None))


def track_all(h: Homotopy, starts: Starts, cfg: TrackConfig | None = None, lo: int = 0, hi: int | None = None,
              device: int = 0, records: Records | None = None, sink=None,
              shard: tuple[int, int, int] | None = None) -> SolutionSet:
    """track_all<R> (tracker.hpp:166-170) on CUDA device `device`: starts [lo, min(count, hi)).

    sink: the ProgressSink (tracker.hpp:70), called with numpy arrays of EVENT_DTYPE (batches of
    StepEvents, tracker.hpp:62-69) while tracking proceeds.  shard: (index, count, block) restricts
    the call to one block-cyclic shard of the range (pp_shard), for multi-GPU partitions."""
    cfg = cfg or TrackConfig.defaults(h.prec)
    count = starts.count
    end = count if hi is None else min(count, hi)
    cap = shard_size(lo, end, shard) if end > lo else 0
    if records is not None:
        if records.prec != h.prec or records.x.shape[1:] != (starts.dim, 2 * LIMBS[h.prec]):
            raise InvalidArgument("track_all: records were allocated for another dimension or precision")
        rec = records
    else:
        rec = Records(max(cap, 1), starts.dim, h.prec)
    c = cfg.to_c()
    st = RunStatsC()
    sh = ShardC(*shard) if shard is not None else None
    errors = []

    def _on_events(ptr, n, _user):
        try:
            buf = (ctypes.c_char * (int(n) * EVENT_DTYPE.itemsize)).from_address(ctypes.addressof(ptr.contents))
            sink(np.frombuffer(buf, dtype=EVENT_DTYPE).copy())
        except BaseException as exc:  # noqa: BLE001 -- re-raised after the call returns
            errors.append(exc)

    cb = EventSinkFn(_on_events) if sink is not None else EventSinkFn()
    _check(lib.pp_track_all_ex(h._h, starts._h, ctypes.byref(c), lo, end if hi is not None else (1 << 64) - 1,
                               ctypes.byref(sh) if sh is not None else None, cb, None, device, ctypes.byref(rec.c),
                               ctypes.byref(st)))
    if errors:
        raise errors[0]
    stats = {f[0]: getattr(st, f[0]) for f in RunStatsC._fields_}
    return rec.solution_set(stats)


def compact_scan(status) -> dict:
    """compact_scan (tracker.hpp:46-54, tracker.cpp:51-65): inclusive prefix scan over
    [status == active], 1-based job labels of the active slots and their slot indices -- the
    paper's compaction step (Table 3).  The device does the same per trip without a
    host round trip (slot refill and tail compaction)."""
    active = (np.asarray(status, dtype=np.int8) == ACTIVE).astype(np.uint32)
    scan = np.cumsum(active, dtype=np.uint32)
    path_idx = np.flatnonzero(active).astype(np.uint32)
    return {"scan": scan, "active_count": int(scan[-1]) if len(scan) else 0,
            "job_idx": np.arange(1, len(path_idx) + 1, dtype=np.uint32), "path_idx": path_idx}


def eval_batch(h: Homotopy, points: np.ndarray, t: np.ndarray, device: int = 0):
    """eval_system_batch (evaldiff.hpp:228-230) on the device: points [B][dim][2L], t [B][L] ->
    (sys [B][n_polys][2L], jac [B][n_polys*dim][2L])."""
    info = h.info
    L = LIMBS[h.prec]
    points = np.ascontiguousarray(points, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64)
    B = points.shape[0]
    sys = np.zeros((B, info["n_polys"], 2 * L))
    jac = np.zeros((B, info["n_polys"] * info["dim"], 2 * L))
    _check(lib.pp_eval_batch(h._h, B, _ptr(points), _ptr(t), _ptr(sys), _ptr(jac), device))
    return sys, jac


def bench_eval(h: Homotopy, seed: int, batch: int, reps: int = 10, device: int = 0):
    """bench-eval (polypath_main.cpp:284-362) on the device: the CLI's points for `seed`, device
    ms per batch evaluation (mean of `reps` launches), and the CLI's FNV-1a checksum (hex)."""
    ms, cs = _dbl(), _u64()
    _check(lib.pp_bench_eval(h._h, seed, batch, reps, device, ctypes.byref(ms), ctypes.byref(cs)))
    return ms.value, f"{cs.value:016x}"


def lsq_batch(prec, a: np.ndarray, b: np.ndarray, device: int = 0):
    """least_squares_solve (linalg.hpp:110-125) batched: a [B][n(col)][n(row)][2L], b [B][n][2L]."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    B, n = a.shape[0], a.shape[1]
    x = np.zeros_like(b)
    ok = np.zeros(B, dtype=np.uint8)
    _check(lib.pp_lsq_batch(_prec(prec), n, B, _ptr(a), _ptr(b), _ptr(x), _ptr(ok), device))
    return x, ok.astype(bool)


def lsq_batch_mn(prec, a: np.ndarray, b: np.ndarray, device: int = 0, factors: bool = False):
    """least_squares_solve / mgs_qr (linalg.hpp:79-125) for m x n systems (m >= n), batched:
    a [B][n(col)][m(row)][2L], b [B][m][2L] -> x [B][n][2L], ok [B] (and with factors=True the
    Q factor [B][n][m][2L] and R packed by columns [B][n(n+1)/2][2L])."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    B, n, m, w = a.shape
    x = np.zeros((B, n, w))
    ok = np.zeros(B, dtype=np.uint8)
    q = np.zeros_like(a) if factors else None
    r = np.zeros((B, n * (n + 1) // 2, w)) if factors else None
    _check(lib.pp_lsq_batch_mn(_prec(prec), m, n, B, _ptr(a), _ptr(b), _ptr(x), _ptr(ok),
                               _ptr(q) if factors else None, _ptr(r) if factors else None, device))
    return (x, ok.astype(bool), q, r) if factors else (x, ok.astype(bool))


def newton_correct(h: Homotopy, t: np.ndarray, x: np.ndarray, cfg: TrackConfig | None = None, device: int = 0):
    """The corrector alone, as PathBatch::set_prediction + newton_correct drive it
    (tracker.hpp:135-136, tracker.cpp:216-274): for each pair (t [B][L], x [B][dim][2L]) up to
    max_newton Newton iterations at that t on the device.  Returns (iterations, corrected,
    singular, last iterates)."""
    cfg = cfg or TrackConfig.defaults(h.prec)
    t = np.ascontiguousarray(t, dtype=np.float64)
    xo = np.ascontiguousarray(x, dtype=np.float64).copy()
    B = len(t)
    it = np.zeros(B, np.uint32)
    co = np.zeros(B, np.uint8)
    sg = np.zeros(B, np.uint8)
    c = cfg.to_c()
    _check(lib.pp_test_newton(h._h, ctypes.byref(c), B, _ptr(t), _ptr(xo), _ptr(it), _ptr(co), _ptr(sg), device))
    return it, co.astype(bool), sg.astype(bool), xo


def fp64_peak(device: int = 0) -> float:
    """measured FP64 pipe operations per second of `device` (DFMA microbenchmark)"""
    v = _dbl()
    _check(lib.pp_fp64_peak(device, ctypes.byref(v)))
    return v.value


def host_arith(prec, op: int, a, b) -> np.ndarray:
    """xprec.cuh host arithmetic (testing hook); op codes as in include/pp200_testing.h"""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.zeros(8)
    _check(lib.pp_test_arith(_prec(prec), op, _ptr(a), _ptr(b), _ptr(out)))
    return out


def to_decimal(prec, limbs) -> str:
    """to_decimal at a level (xprec_io.cpp:31-108): 17 / 32 / 64 significant digits."""
    a = np.zeros(4)
    a[: len(limbs)] = limbs
    buf = ctypes.create_string_buffer(128)
    _check(lib.pp_to_decimal(_prec(prec), _ptr(a), buf, 128))
    return buf.value.decode()


def parse_decimal(prec, s: str) -> np.ndarray:
    out = np.zeros(4)
    _check(lib.pp_test_parse_decimal(_prec(prec), s.encode(), _ptr(out)))
    return out[: LIMBS[_pname(prec)]]


__all__ = [
    "System", "Starts", "Homotopy", "TrackConfig", "SolutionSet", "Records", "parse_system", "cyclic_system",
    "random_gamma", "total_degree_start", "explicit_starts", "load_start_data", "make_homotopy", "track_all",
    "eval_batch", "lsq_batch", "InvalidArgument", "ParseError", "CudaError", "PRECISIONS", "LIMBS", "REASONS",
]
