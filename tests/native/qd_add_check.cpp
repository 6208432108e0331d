// Bitwise check of the network-merge quad-double addition (qdi::add_i) against the step-by-step
// merge (qdi::add_seq_i, the restatement of xprec.hpp:325-382 that the GPU parity suite pins to the
// reference) on random, structured and adversarial operands.  Built and run by
// tests/test_host.py::test_qd_add_network_matches_sequential_merge.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>

#include "xprec.cuh"

using pp::qd_t;

static uint64_t bits(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}
static bool same(const qd_t& x, const qd_t& y) {
  return bits(x.c0) == bits(y.c0) && bits(x.c1) == bits(y.c1) && bits(x.c2) == bits(y.c2) && bits(x.c3) == bits(y.c3);
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 2000000;
  std::mt19937_64 rng(20261017);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  std::uniform_int_distribution<int> E(-60, 60), pick(0, 15);
  const double specials[] = {0.0, -0.0, 1.0, -1.0, 0.5, std::ldexp(1.0, -1074), -std::ldexp(1.0, -1074),
                             std::ldexp(1.0, -1022), std::numeric_limits<double>::infinity(),
                             -std::numeric_limits<double>::infinity(), std::numeric_limits<double>::quiet_NaN(),
                             std::ldexp(1.0, 1023)};
  auto rnd_qd = [&](int e) {
    // a renormalised value: a sum of four doubles of decreasing magnitude
    qd_t x = pp::qd_make(std::ldexp(U(rng), e));
    for (int l = 1; l < 4; ++l) x = pp::qdi::add_seq_i(x, pp::qd_make(std::ldexp(U(rng), e - 53 * l - (int)(rng() % 8))));
    return x;
  };
  auto operand = [&](const qd_t& other) -> qd_t {
    switch (pick(rng)) {
      case 0: return pp::qd_make(std::ldexp(U(rng), E(rng)));                    // one limb
      case 1: return pp::rneg(other);                                             // exact cancellation
      case 2: { qd_t o = other; o.c3 = -o.c3; o.c2 = 0.0; return o; }             // partial cancellation
      case 3: return pp::qd_make(specials[rng() % 12]);
      case 4: { qd_t o{specials[rng() % 12], specials[rng() % 12], specials[rng() % 12], specials[rng() % 12]}; return o; }
      case 5: { qd_t o{U(rng), U(rng), U(rng), U(rng)}; return o; }                // unordered limbs
      case 6: { qd_t o = other; o.c1 = -o.c1; return o; }                         // equal magnitudes
      case 7: { qd_t o{other.c0, -other.c0, 0.0, -0.0}; return o; }
      case 8: return pp::qdi::mul_i(rnd_qd(E(rng) / 4), rnd_qd(E(rng) / 4));
      case 9: { qd_t o = other; o.c0 = std::ldexp(o.c0, 1); return o; }
      default: return rnd_qd(E(rng));
    }
  };
  long bad = 0, fast = 0;
  for (long i = 0; i < n; ++i) {
    const qd_t a = (i & 3) ? rnd_qd(E(rng)) : operand(rnd_qd(E(rng)));
    const qd_t b = operand(a);
    const qd_t x = (i & 1) ? pp::qdi::add_i(a, b) : pp::qdi::add_i(b, a);
    const qd_t y = (i & 1) ? pp::qdi::add_seq_i(a, b) : pp::qdi::add_seq_i(b, a);
    if (!same(x, y)) {
      if (++bad <= 5)
        std::printf("MISMATCH a=(%a %a %a %a) b=(%a %a %a %a)\n", a.c0, a.c1, a.c2, a.c3, b.c0, b.c1, b.c2, b.c3);
    }
    fast += std::fabs(a.c0) >= std::fabs(a.c1) && std::fabs(a.c1) >= std::fabs(a.c2) && std::fabs(a.c2) >= std::fabs(a.c3) &&
            std::fabs(b.c0) >= std::fabs(b.c1) && std::fabs(b.c1) >= std::fabs(b.c2) && std::fabs(b.c2) >= std::fabs(b.c3);
  }
  std::printf("qd add: %ld operand pairs, %ld through the network merge, %ld mismatches\n", n, fast, bad);
  return bad ? 1 : 0;
}
