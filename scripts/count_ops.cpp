// Counts binary64 operations of the level arithmetic (xprec.cuh, host build) per operation,
// averaged over random operands of tracker-like magnitude.  Feeds the work model
// (paper_1505_00383_b200/work.py OPS table).
//   g++ -O1 -std=c++20 -ffp-contract=off -DPP_COUNT_OPS -I paper_1505_00383_b200/csrc \
//       scripts/count_ops.cpp -o /tmp/count_ops && /tmp/count_ops
#include <cstdio>
#include <random>

#include "xprec.cuh"

unsigned long long pp_op_count = 0;

template <class R>
R random_level(std::mt19937_64& g, int L) {
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::uniform_int_distribution<int> e(-3, 3);
  R v = pp::rfrom<R>(0.0);
  double x = u(g) * std::ldexp(1.0, e(g));
  for (int l = 0; l < L; ++l) {
    pp::level<R>::set(v, l, x);
    x = x * u(g) * 0x1p-53;
  }
  return v;
}

template <class R>
void run(const char* name, int L) {
  std::mt19937_64 g(42);
  const int N = 100000;
  unsigned long long c[5] = {0, 0, 0, 0, 0};
  for (int i = 0; i < N; ++i) {
    R a = random_level<R>(g, L), b = random_level<R>(g, L);
    unsigned long long s = pp_op_count;
    volatile R r1 = pp::radd(a, b);
    c[0] += pp_op_count - s;
    s = pp_op_count;
    volatile R r2 = pp::rmul(a, b);
    c[1] += pp_op_count - s;
    s = pp_op_count;
    volatile R r3 = pp::rmuld(a, 1.5);
    c[2] += pp_op_count - s;
    s = pp_op_count;
    volatile R r4 = pp::rdiv(a, b);
    c[3] += pp_op_count - s;
    s = pp_op_count;
    volatile R r5 = pp::rsqrt(pp::rabs(a));
    c[4] += pp_op_count - s;
    (void)r1, (void)r2, (void)r3, (void)r4, (void)r5;
  }
  std::printf("%s: add=%.1f mul=%.1f muld=%.1f div=%.1f sqrt=%.1f\n", name, double(c[0]) / N, double(c[1]) / N,
              double(c[2]) / N, double(c[3]) / N, double(c[4]) / N);
}

int main() {
  run<double>("d", 1);
  run<pp::dd_t>("dd", 2);
  run<pp::qd_t>("qd", 4);
}
