"""Writes the benchmark systems the reference does not ship in its .sys format:

* katsura12.sys -- katsura-12 (13 unknowns x0..x12):  x0 + 2*sum_{i=1..12} x_i - 1 and, for
  m = 0..11, sum_{l=-12..12} x_|l| * x_|m-l| - x_m with terms whose index exceeds 12 dropped;
  Bezout number 2^12 = 4096.
* rand32.sys is written by scripts/gen_rand32.cpp (std::mt19937_64(12345), the generator
  SURVEY.md 8(d) names).

The files are committed under tests/data so the oracle and the GPU read identical text.
"""

import os
from collections import OrderedDict


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


if __name__ == "__main__":
    with open(os.path.join(OUT, "katsura12.sys"), "w") as fh:
        fh.write(katsura())
    print("wrote katsura12.sys (rand32.sys: scripts/gen_rand32.cpp)")
