// Writes tests/data/rand32.sys, the synthetic sparse system of SURVEY.md 8(d): n = 32 unknowns,
// 16 quadratic and 16 linear polynomials (Bezout number 2^16 = 65,536), each with 8 random
// monomial terms plus a constant, the first term at full degree, coefficients uniform in
// [-1, 1]^2, all drawn from std::mt19937_64(12345).  Monomials: the first term multiplies `deg`
// variables drawn uniformly (with repetition, so x_i^2 can occur); the others draw a degree in
// [1, deg] and that many variables; a monomial already in the polynomial is redrawn.
// Coefficients print with 17 significant digits, so every reader parses the same doubles.
//
//   g++ -O2 -std=c++17 scripts/gen_rand32.cpp -o /tmp/gen_rand32 && /tmp/gen_rand32 > tests/data/rand32.sys
#include <cstdio>
#include <map>
#include <random>
#include <set>
#include <string>
#include <vector>

int main() {
  const unsigned n = 32;
  std::mt19937_64 rng(12345);
  std::uniform_real_distribution<double> coef(-1.0, 1.0);
  std::printf("%u;\n", n);
  for (unsigned i = 0; i < n; ++i) {
    const unsigned deg = i < n / 2 ? 2 : 1;
    std::set<std::map<unsigned, unsigned>> seen;
    std::string line;
    unsigned terms = 0;
    while (terms < 8) {
      const unsigned d = terms == 0 ? deg : 1 + static_cast<unsigned>(rng() % deg);
      std::map<unsigned, unsigned> mono;
      for (unsigned k = 0; k < d; ++k) ++mono[static_cast<unsigned>(rng() % n)];
      if (!seen.insert(mono).second) continue;
      const double re = coef(rng), im = coef(rng);
      char buf[96];
      std::snprintf(buf, sizeof buf, "(%.17g,%.17g)", re, im);
      if (terms) line += " + ";
      line += buf;
      for (const auto& [v, e] : mono) {
        line += "*x" + std::to_string(v);
        if (e > 1) line += "^" + std::to_string(e);
      }
      ++terms;
    }
    char buf[96];
    const double re = coef(rng), im = coef(rng);
    std::snprintf(buf, sizeof buf, " + (%.17g,%.17g)", re, im);
    line += buf;
    std::printf("%s;\n", line.c_str());
  }
  return 0;
}
