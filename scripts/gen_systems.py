"""Writes the benchmark systems the reference does not ship in its .sys format:

* katsura12.sys -- katsura-12 (13 unknowns x0..x12):  x0 + 2*sum_{i=1..12} x_i - 1 and, for
  m = 0..11, sum_{l=-12..12} x_|l| * x_|m-l| - x_m with terms whose index exceeds 12 dropped;
  Bezout number 2^12 = 4096.
* rand32.sys -- synthetic sparse n = 32: 16 quadratic + 16 linear polynomials, 8 random terms plus
  a constant each, the first term at full degree, coefficients uniform in [-1, 1]^2 (numpy
  PCG64 seed 12345), written with 17 significant digits; Bezout 2^16 = 65536.

The files are committed under tests/data so the oracle and the GPU read identical text.
"""

import os
from collections import OrderedDict

import numpy as np

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "data")


def mono_text(mono):
    return "*".join(f"x{v}" + (f"^{e}" if e > 1 else "") for v, e in sorted(mono.items()))


def katsura(n=12):
    polys = []
    lin = ["x0"] + [f"2*x{i}" for i in range(1, n + 1)]
    polys.append(" + ".join(lin) + " - 1")
    for m in range(n):
        acc = OrderedDict()
        for l in range(-n, n + 1):
            a, b = abs(l), abs(m - l)
            if a > n or b > n:
                continue
            key = tuple(sorted({a: 0, b: 0}.keys()))
            mono = {}
            mono[a] = mono.get(a, 0) + 1
            mono[b] = mono.get(b, 0) + 1
            k = tuple(sorted(mono.items()))
            acc[k] = acc.get(k, 0) + 1
        terms = []
        for k, c in acc.items():
            t = mono_text(dict(k))
            terms.append(t if c == 1 else f"{c}*{t}")
        polys.append(" + ".join(terms) + f" - x{m}")
    return f"{n + 1};\n" + "".join(p + ";\n" for p in polys)


def rand32(seed=12345, n=32):
    rng = np.random.default_rng(seed)
    polys = []
    for i in range(n):
        deg = 2 if i < n // 2 else 1
        terms = []
        seen = set()
        while len(terms) < 8:
            if not terms:
                # first term at full degree
                vs = rng.choice(n, size=deg, replace=deg == 2)
            else:
                d = int(rng.integers(1, deg + 1))
                vs = rng.choice(n, size=d, replace=True)
            mono = {}
            for v in vs:
                mono[int(v)] = mono.get(int(v), 0) + 1
            key = tuple(sorted(mono.items()))
            if key in seen or sum(mono.values()) > deg:
                continue
            seen.add(key)
            re, im = rng.uniform(-1, 1, 2)
            terms.append(f"({re:.17g},{im:.17g})*{mono_text(mono)}")
        re, im = rng.uniform(-1, 1, 2)
        terms.append(f"({re:.17g},{im:.17g})")
        polys.append(" + ".join(terms))
    return f"{n};\n" + "".join(p + ";\n" for p in polys)


if __name__ == "__main__":
    with open(os.path.join(OUT, "katsura12.sys"), "w") as fh:
        fh.write(katsura())
    with open(os.path.join(OUT, "rand32.sys"), "w") as fh:
        fh.write(rand32())
    print("wrote katsura12.sys, rand32.sys")
