"""Golden checksums of the reference's bench-eval (polypath_main.cpp:284-362): the CLI's
splitmix64 points and t for a seed, eval_system_batch of the UNMODIFIED reference build
(oracle/_ref), FNV-1a over ws.sys.raw() then ws.jac.raw() (planar [row][plane][batch]).  The CLI
itself cannot be built offline (CLI11 is not vendored), so its point stream and hash are restated
here and the evaluation is the reference library's.

    python tests/golden/make_bench_eval.py   ->   tests/golden/bench_eval.json
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

M64 = (1 << 64) - 1
CASES = [("cyclic5", "d", 7, 10), ("cyclic10", "dd", 1, 64), ("cyclic10", "qd", 3, 20), ("katsura12", "dd", 5, 33)]


def units(seed: int, count: int):
    state = (seed * 0x9E3779B97F4A7C15 + 0x243F6A8885A308D3) & M64
    out = []
    for _ in range(count):
        state = (state + 0x9E3779B97F4A7C15) & M64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        z ^= z >> 31
        out.append(2.0 * (float(z >> 11) * 2.0 ** -53) - 1.0)
    return out


def fnv1a(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & M64
    return h


def reference_checksum(text: str, prec: str, seed: int, batch: int) -> str:
    L = O.LIMBS[prec]
    dim = int(text.strip().split(";")[0].split()[0])
    u = units(seed, batch * (2 * dim + 1))
    pts = np.zeros((batch, dim, 2 * L))
    t = np.zeros((batch, L))
    k = 0
    for j in range(batch):
        for v in range(dim):
            pts[j, v, 0], pts[j, v, L] = u[k], u[k + 1]
            k += 2
        t[j, 0] = 0.5 * (u[k] + 1.0)
        k += 1
    gam = O.ref_random_gamma(1)
    g = np.zeros(2 * L)
    g[0], g[L] = gam.real, gam.imag
    sys_, jac = O.ref_eval(text, prec, g, pts, t)
    # user layout [batch][row][plane] -> PlanarBlock raw [row][plane][batch]
    raw = np.concatenate([np.transpose(sys_, (1, 2, 0)).ravel(), np.transpose(jac, (1, 2, 0)).ravel()])
    return f"{fnv1a(raw.astype('<f8').tobytes()):016x}"


def main():
    out = []
    for system, prec, seed, batch in CASES:
        with open(os.path.join(ROOT, "tests", "data", system + ".sys")) as fh:
            text = fh.read()
        cs = reference_checksum(text, prec, seed, batch)
        out.append({"system": system, "prec": prec, "seed": seed, "batch": batch, "gamma_seed": 1, "checksum": cs})
        print(out[-1], flush=True)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "bench_eval.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
