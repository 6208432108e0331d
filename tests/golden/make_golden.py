"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED reference library
(oracle/_ref/libppref.so, built from /root/reference/proj/src by oracle/Makefile) in this
container.  The fixtures pin both the C oracle (oracle/oracle.c) and the CUDA path; they are
committed so that the GPU box (where /root/reference does not exist) can check against them.

    python tests/golden/make_golden.py
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DATA = os.path.join(ROOT, "tests", "data")
SQUARE_F = "1; x0^2 - 4;"
SQUARE_G = "1; x0^2 - 1;"
CYC3 = O.ref_cyclic_text(3) if O.ref is not None else None


def gamma_limbs(g: complex, prec: str):
    L = O.LIMBS[prec]
    a = np.zeros(2 * L)
    a[0], a[L] = g.real, g.imag
    return a


def save_track(name, text, prec, gamma_seed, lo, hi, cfg=None, g_text=None, starts_text=None):
    gam = O.ref_random_gamma(gamma_seed)
    r = O.ref_track(text, prec, gam, cfg=cfg, lo=lo, hi=hi, g_text=g_text, starts_text=starts_text,
                    workers=8, batch=512)
    np.savez_compressed(os.path.join(HERE, f"track_{name}.npz"), prec=prec, gamma_seed=gamma_seed, lo=lo, hi=hi,
                        cfg=repr(cfg or {}), **{k: v for k, v in r.items() if k not in ("wall_ms",)})
    counts = {"converged": int(np.sum(r["status"] == 1))}
    print(f"track_{name}: {len(r['status'])} paths, {counts}, {r['wall_ms']:.0f} ms", flush=True)


def save_eval(name, text, prec, seed, batch=16):
    rng = np.random.default_rng(seed)
    dim = int(text.split(";")[0])
    L = O.LIMBS[prec]
    pts = np.zeros((batch, dim, 2 * L))
    pts[:, :, 0] = rng.uniform(-1.5, 1.5, (batch, dim))
    pts[:, :, L] = rng.uniform(-1.5, 1.5, (batch, dim))
    for l in range(1, L):  # nonzero lower limbs exercise the full extended arithmetic
        pts[:, :, l] = pts[:, :, l - 1] * rng.uniform(-1, 1, (batch, dim)) * 2.0 ** -54
        pts[:, :, L + l] = pts[:, :, L + l - 1] * rng.uniform(-1, 1, (batch, dim)) * 2.0 ** -54
    t = np.zeros((batch, L))
    t[:, 0] = rng.uniform(0, 1, batch)
    t[0, 0], t[1, 0] = 0.0, 1.0
    gl = gamma_limbs(O.ref_random_gamma(1), prec)
    sys_, jac = O.ref_eval(text, prec, gl, pts, t)
    np.savez_compressed(os.path.join(HERE, f"eval_{name}.npz"), prec=prec, points=pts, t=t, gamma=gl, sys=sys_, jac=jac)
    print(f"eval_{name}: {batch} points")


def save_lsq(name, prec, n, seed, batch=32):
    rng = np.random.default_rng(seed)
    L = O.LIMBS[prec]
    a = np.zeros((batch, n, n, 2 * L))
    b = np.zeros((batch, n, 2 * L))
    a[..., 0] = rng.standard_normal((batch, n, n))
    a[..., L] = rng.standard_normal((batch, n, n))
    b[..., 0] = rng.standard_normal((batch, n))
    b[..., L] = rng.standard_normal((batch, n))
    for l in range(1, L):
        a[..., l] = a[..., l - 1] * rng.uniform(-1, 1, a.shape[:-1]) * 2.0 ** -54
        a[..., L + l] = a[..., L + l - 1] * rng.uniform(-1, 1, a.shape[:-1]) * 2.0 ** -54
    # rank-deficient and ill-conditioned members: duplicated column, zero column, near-dependent column
    if n >= 2:
        a[1, 1] = a[1, 0]
    a[2, n - 1] = 0.0
    if n > 2:
        a[3, 2] = a[3, 0] * 0.5 + a[3, 1] * 1e-7
    x, ok = O.ref_lsq(prec, a, b)
    np.savez_compressed(os.path.join(HERE, f"lsq_{name}.npz"), prec=prec, a=a, b=b, x=x, ok=ok)
    print(f"lsq_{name}: {batch} systems, {int(ok.sum())} ok")


def main(force=False):
    assert O.ref is not None, "build the reference first: make -C oracle ref"
    rd = lambda name: open(os.path.join(DATA, name)).read()  # noqa: E731
    c5, c10, c8 = rd("cyclic5.sys"), rd("cyclic10.sys"), O.ref_cyclic_text(8)
    k12, r32 = rd("katsura12.sys"), rd("rand32.sys")
    c5g, c5s = rd("cyclic5_start.sys"), rd("cyclic5_starts.txt")
    jobs = []
    for prec in ("d", "dd", "qd"):
        jobs.append((f"eval_cyclic5_{prec}", lambda p=prec: save_eval(f"cyclic5_{p}", c5, p, 5)))
        jobs.append((f"eval_cyclic10_{prec}", lambda p=prec: save_eval(f"cyclic10_{p}", c10, p, 10)))
        for n in (1, 5, 10, 13):
            jobs.append((f"lsq_n{n}_{prec}", lambda p=prec, n=n: save_lsq(f"n{n}_{p}", p, n, 100 + n)))
    tracks = [
        ("square_d", SQUARE_F, "d", 1, 0, 2, None, dict(g_text=SQUARE_G, starts_text="1,0\n-1,0\n")),
        ("cyclic3_dd", CYC3, "dd", 3, 0, 6, None, {}),
        ("cyclic5_d", c5, "d", 1, 0, 120, None, {}),
        ("cyclic5_dd", c5, "dd", 1, 0, 120, None, {}),
        ("cyclic5_qd", c5, "qd", 1, 0, 8, None, {}),
        ("cyclic5_dd_seed101", c5, "dd", 101, 0, 120, None, {}),
        ("cyclic5_file_dd", c5, "dd", 1, 0, 120, None, dict(g_text=c5g, starts_text=c5s)),
        ("cyclic10_d", c10, "d", 1, 0, 512, None, {}),
        ("cyclic10_dd", c10, "dd", 1, 0, 128, None, {}),
        ("cyclic10_dd_far", c10, "dd", 1, 1000000, 1000032, None, {}),
        ("cyclic5_d_tight", c5, "d", 1, 0, 120, {"max_newton": 2, "h_init": 0.1, "max_steps": 40}, {}),
        ("cyclic8_d", c8, "d", 1, 0, 1024, None, {}),
        ("cyclic8_dd", c8, "dd", 1, 0, 64, None, {}),
        ("katsura12_d", k12, "d", 1, 0, 256, None, {}),
        ("katsura12_dd", k12, "dd", 1, 0, 32, None, {}),
        ("katsura12_qd_mn4", k12, "qd", 1, 0, 4, {"max_newton": 4}, {}),
        ("rand32_d", r32, "d", 1, 0, 128, None, {}),
        ("rand32_dd", r32, "dd", 1, 0, 8, None, {}),
        ("rand32_qd", r32, "qd", 1, 0, 2, None, {}),
        ("cyclic8_qd", c8, "qd", 1, 0, 4, None, {}),
        ("cyclic10_qd", c10, "qd", 1, 2000000, 2000002, None, {}),
    ]
    for name, text, prec, seed, lo, hi, cfg, kw in tracks:
        jobs.append((f"track_{name}", lambda a=(name, text, prec, seed, lo, hi, cfg, kw):
                     save_track(a[0], a[1], a[2], a[3], a[4], a[5], cfg=a[6], **a[7])))
    for fname, job in jobs:
        if force or not os.path.exists(os.path.join(HERE, fname + ".npz")):
            job()


if __name__ == "__main__":
    main(force="--force" in sys.argv)
