// homotopy.cpp -- total-degree start systems and start-solution tables.
//
// Roots of unity are seeded from double cos/sin and polished by 0/2/3 Newton steps on x^d = 1 at
// the run level, and start tuples are enumerated lexicographically with the last variable
// fastest, as in reference homotopy.cpp:42-113.  The tables are uploaded once; the device
// generates start index -> start point itself.

#include <cmath>

#include "host.hpp"

namespace pp {

namespace {

template <class R>
void unity_roots(uint32_t d, std::vector<double>& out) {
  constexpr int L = level<R>::L;
  const int polish = L == 1 ? 0 : (L == 2 ? 2 : 3);
  const cx<R> one = cone<R>();
  for (uint32_t j = 0; j < d; ++j) {
    double theta = 2.0 * M_PI * static_cast<double>(j) / static_cast<double>(d);
    cx<R> x{rfrom<R>(std::cos(theta)), rfrom<R>(std::sin(theta))};
    for (int it = 0; it < polish; ++it) {
      cx<R> xp = one;  // x^(d-1)
      for (uint32_t e = 1; e < d; ++e) xp = cmul(xp, x);
      cx<R> fx = csub(cmul(xp, x), one);
      cx<R> fpx = cmulr(xp, rfrom<R>(static_cast<double>(d)));
      x = csub(x, cdiv(fx, fpx));
    }
    for (int l = 0; l < L; ++l) out.push_back(level<R>::get(x.re, l));
    for (int l = 0; l < L; ++l) out.push_back(level<R>::get(x.im, l));
  }
}

}  // namespace

void Starts::solution(uint64_t index, double* x) const {
  const size_t w = 2 * L;
  if (!total_degree) {
    const double* src = explicit_x.data() + index * dim * w;
    std::copy(src, src + dim * w, x);
    return;
  }
  uint64_t rem = index;
  for (size_t i = dim; i-- > 0;) {
    const uint32_t d = degrees[i];
    const double* r = roots.data() + (root_off[i] + rem % d) * w;
    std::copy(r, r + w, x + i * w);
    rem /= d;
  }
}

std::pair<System, Starts> total_degree_start(const System& f, int prec) {
  if (f.dim != f.polys.size()) throw InvalidArgument("total_degree_start: system must be square");
  Starts sd;
  sd.prec = prec;
  sd.L = prec == 0 ? 1 : (prec == 1 ? 2 : 4);
  sd.dim = f.dim;
  sd.total_degree = true;
  sd.count = 1;
  System g;
  g.dim = f.dim;
  uint32_t off = 0;
  for (uint32_t i = 0; i < f.dim; ++i) {
    const uint32_t d = f.degrees[i];
    if (d == 0) throw InvalidArgument("total_degree_start: zero-degree polynomial");
    sd.degrees.push_back(d);
    sd.root_off.push_back(off);
    off += d;
    switch (prec) {
      case 0: unity_roots<double>(d, sd.roots); break;
      case 1: unity_roots<dd_t>(d, sd.roots); break;
      default: unity_roots<qd_t>(d, sd.roots); break;
    }
    sd.count *= d;
    Monomial m;
    m.factors.emplace_back(i, d);
    g.polys.push_back({Term{cqd{qd_make(1.0), qd_make(0.0)}, std::move(m)},
                       Term{cqd{qd_make(-1.0), qd_make(0.0)}, Monomial{}}});
  }
  g.refresh_degrees();
  return {std::move(g), std::move(sd)};
}

}  // namespace pp
