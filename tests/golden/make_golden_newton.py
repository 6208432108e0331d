"""Golden corrector runs: the reference's PathBatch::set_prediction + newton_correct
(tracker.hpp:135-136, tracker.cpp:216-274; the hook test_tracker.cpp:121-196 and acceptance
criterion 9 use) on chosen (t, x) pairs -- on-path, nearby, hopeless and rank-deficient
predictions -- from the UNMODIFIED reference build (oracle/_ref).

    python tests/golden/make_golden_newton.py
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DATA = os.path.join(ROOT, "tests", "data")
SQUARE_F, SQUARE_G = "1; x0^2 - 4;", "1; x0^2 - 1;"


def widen(x, L):
    """[B][dim][2] doubles -> [B][dim][2L] limbs"""
    out = np.zeros(x.shape[:-1] + (2 * L,))
    out[..., 0], out[..., L] = x[..., 0], x[..., 1]
    return out


def glimbs(g, L):
    a = np.zeros(2 * L)
    a[0], a[L] = g.real, g.imag
    return a


def square_case(prec):
    L = O.LIMBS[prec]
    xs = np.sqrt(1.0 + 3.0 * 0.5)
    t = [0.16, 1.0, 1.0, 0.5, 0.5, 0.5, 0.5]
    x = [np.sqrt(1.48), 2.1, 2.0001, complex(250, 40), xs + 1e-2, xs + 1e-9, xs + 1e-5]
    tt = np.zeros((len(t), L))
    tt[:, 0] = t
    xx = widen(np.array([[[complex(v).real, complex(v).imag]] for v in x]), L)
    return SQUARE_F, SQUARE_G, tt, xx, glimbs(1.0, L)


def near_starts_case(name, prec, count, seed, t_value):
    """perturbed total-degree start solutions at a small t, plus a few hopeless points and the
    origin (rank-deficient Jacobian)"""
    L = O.LIMBS[prec]
    text = open(os.path.join(DATA, name + ".sys")).read()
    dim = int(text.split(";")[0])
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, 1000, count)
    xs = np.stack([O.ref_td_solution(text, prec, int(i), dim) for i in idx])
    scale = 10.0 ** -rng.integers(3, 12, count)[:, None]  # from 1e-3 (rejected) to 1e-11 (certified)
    xs[..., 0] += rng.normal(0, 1, xs[..., 0].shape) * scale
    xs[..., L] += rng.normal(0, 1, xs[..., L].shape) * scale
    xs[count - 3] *= 40.0
    xs[count - 2, :, 0] += 3.0
    xs[count - 1] = 0.0
    tt = np.zeros((count, L))
    tt[:, 0] = 0.0  # t = 0: the perturbed start solutions of gamma*g
    tt[count // 2:, 0] = t_value
    return text, None, tt, xs, glimbs(O.ref_random_gamma(1), L)


CASES = []
for prec in ("d", "dd", "qd"):
    CASES.append((f"square_{prec}", prec, square_case(prec), {}))
    CASES.append((f"square_{prec}_mn2", prec, square_case(prec), {"max_newton": 2}))
    CASES.append((f"cyclic5_{prec}", prec, near_starts_case("cyclic5", prec, 24, 7, 0.01), {}))
CASES.append(("cyclic10_dd", "dd", near_starts_case("cyclic10", "dd", 24, 11, 0.02), {}))

if __name__ == "__main__":
    out = {}
    for name, prec, (f, g, t, x, gl), cfg in CASES:
        it, co, xo, rounds = O.ref_newton(f, prec, gl, t, x, cfg=cfg, g_text=g)
        out[name] = dict(prec=prec, f=f, g=g or "", gamma=gl, cfg=repr(cfg), t=t, x=x, iters=it, corrected=co,
                         x_out=xo, rounds=rounds)
        print(name, "iterations", it.tolist(), "corrected", co.astype(int).tolist(), "rounds", rounds)
    flat = {f"{n}__{k}": v for n, d in out.items() for k, v in d.items()}
    np.savez_compressed(os.path.join(HERE, "newton_cases.npz"), names=np.array(list(out)), **flat)
