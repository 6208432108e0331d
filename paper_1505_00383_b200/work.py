"""Algorithmic work model of the tracker's hot path, computed from the plan.

Unit of work: one path Newton iteration = one evaluation of H and dH/dx (evaldiff.cpp:259-374)
plus one least-squares solve (linalg.hpp:79-125).  Work is counted in binary64 operations of
the reference's arithmetic (xprec.hpp / complex.hpp): every +, -, *, fma, /, sqrt on a double
counts 1, so a double-double addition is 20 ops, a product 11, a product by a double 6, and a
complex double-double product 84 (4 products + 2 additions).  Quad-double costs are
data-dependent (merge-based addition, renormalisation branches); their per-operation counts are
averages measured with the op-counting host build (scripts/count_ops.py) and recorded here.

Bytes: the compulsory HBM traffic of one iteration in the multi-kernel design -- the Jacobian and
right-hand side written by the evaluation and read by the solver, Q written back, R/y scratch,
x read/written -- is what `bytes_per_iteration` returns; the FP64-operation intensity of every
precision is far above the B200 ridge point, so the FP64 pipe is the bound.
"""

from __future__ import annotations

# binary64 operations per level operation: add, mul, mul-by-double, div, sqrt, compare-free
OPS = {
    "d": dict(add=1, mul=1, muld=1, div=1, sqrt=1),
    "dd": dict(add=20, mul=11, muld=6, div=68, sqrt=42),
    # measured averages (scripts/count_ops.cpp, 10^5 random operands of tracker-like magnitude)
    "qd": dict(add=94, mul=180, muld=64, div=662, sqrt=2205),
}


def _c(prec):
    o = OPS[prec]
    cmul = 4 * o["mul"] + 2 * o["add"]
    cadd = 2 * o["add"]
    cmulr = 2 * o["mul"]
    cmuld = 2 * o["muld"]
    abs2 = 2 * o["mul"] + o["add"]
    cabs = abs2 + o["sqrt"]
    # Smith division: |re| >= |im| branch: 3 div + 3 mul + 3 add
    cdiv = 3 * o["div"] + 3 * o["mul"] + 3 * o["add"]
    return o, cmul, cadd, cmulr, cmuld, abs2, cabs, cdiv


def eval_ops(info: dict, prec: str) -> int:
    """binary64 ops of one evaluation (coefficient + monomial + sum stages, fused)."""
    o, cmul, cadd, cmulr, cmuld, abs2, cabs, cdiv = _c(prec)
    n_terms = info["n_terms"]
    w = 0
    w += n_terms * (4 * o["mul"] + 2 * o["add"])      # c = cs*(1-t) + ct*t
    w += info["cmul_steps"] * cmul                     # Speelpenning + common-factor products
    w += n_terms * (cmul + cadd)                       # sys += c*value (constants: add only)
    w += info["jac_terms"] * (cmul + cadd)             # jac += c*d_j
    w += info["jac_scaled"] * cmuld                    # exponent scaling
    w += info["n_polys"] * (cabs + 1)                  # residual norms
    return w


def lsq_ops(n: int, prec: str) -> int:
    """binary64 ops of one two-pass MGS least-squares solve of an n x n complex system."""
    o, cmul, cadd, cmulr, cmuld, abs2, cabs, cdiv = _c(prec)
    w = n * n * (abs2 + o["add"]) + n * o["sqrt"] + o["mul"]          # column norms, tolerance
    proj = n * (cmul + cadd) + cadd + n * (cmul + cadd)                 # dot, R update, axpy
    w += 2 * (n * (n - 1) // 2) * proj                                  # two passes, i < k
    w += n * (n * (abs2 + o["add"]) + o["sqrt"] + o["div"])             # r_kk, 1/r_kk
    w += n * n * cmulr + n * n * (cmul + cadd)                          # normalise, y = Q^H b
    w += (n * (n - 1) // 2) * (cmul + cadd) + n * cdiv                  # back substitution
    w += n * (cadd + 2 * (cabs + 1))                                    # x += dx, norms
    return w


def bytes_per_iteration(n: int, prec: str) -> int:
    """compulsory global-memory bytes of one evaluation + solve (one slot)."""
    L = {"d": 1, "dd": 2, "qd": 4}[prec]
    c = 16 * L  # bytes per complex value
    nJ, nR = n * n, n * (n + 1) // 2
    # eval: x read, J and b written; lsq: J read, Q written, R/y written+read, b read, x read+written
    return c * (n + nJ + n) + c * (nJ + nJ + 2 * nR + 2 * n + n + 2 * n)


def path_work(info: dict, prec: str, evals: int, solves: int) -> dict:
    """total algorithmic ops of a run with `evals` evaluations and `solves` solves"""
    n = info["dim"]
    we, wl = eval_ops(info, prec), lsq_ops(n, prec)
    return {"eval_ops": we, "lsq_ops": wl, "total_ops": evals * we + solves * wl,
            "eval_total": evals * we, "lsq_total": solves * wl}
