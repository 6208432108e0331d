// host.hpp -- host-side data model of the B200 tracker: polynomial systems, the evaluation plan
// (SoA instruction tables uploaded to the device), start data and homotopies.
//
// The host keeps the reference's drop-in API shape (parse_system / cyclic_system / make_homotopy /
// total_degree_start / load_start_data / track_all, reference polysys.hpp:67-99,
// homotopy.hpp:16-68, tracker.hpp:166-170); everything numeric that crosses into a kernel is
// flattened into plain arrays of binary64 limbs here.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "xprec.cuh"

namespace pp {

using cqd = cx<qd_t>;

// (variable, exponent) pairs sorted by variable; empty = constant (polysys.hpp:23-35)
struct Monomial {
  std::vector<std::pair<uint32_t, uint32_t>> factors;
  uint32_t degree() const {
    uint32_t d = 0;
    for (const auto& f : factors) d += f.second;
    return d;
  }
  bool operator==(const Monomial& o) const { return factors == o.factors; }
  bool operator<(const Monomial& o) const { return factors < o.factors; }
};

struct Term {
  cqd coeff;
  Monomial mono;
};

struct System {
  uint32_t dim = 0;
  std::vector<std::vector<Term>> polys;
  std::vector<uint32_t> degrees;
  void refresh_degrees();
  uint64_t monomial_count() const;
};

struct ParseFailure : std::runtime_error {
  size_t line, col;
  ParseFailure(const std::string& m, size_t l, size_t c) : std::runtime_error(m), line(l), col(c) {}
};

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

// decimal text -> level (xprec_io.cpp:121-193); false on malformed input
bool parse_decimal_qd(std::string_view s, qd_t& out);
bool parse_decimal_dd(std::string_view s, dd_t& out);
bool parse_decimal_d(std::string_view s, double& out);
std::string to_decimal_qd(qd_t x);
std::string to_decimal_dd(dd_t x);
std::string to_decimal_d(double x);

System parse_system(std::string_view text);
std::string print_system(const System& s);
System cyclic_system(uint32_t n);

// lines of "re,im, re,im, ..." (parse_solutions, polysys.cpp:381-425)
std::vector<std::vector<cqd>> parse_solutions(std::string_view text, uint32_t dim);

// splitmix64-based e^{i theta} (homotopy.cpp:24-40)
void random_gamma(uint64_t seed, double& re, double& im);

// ---------------------------------------------------------------------------------------------
// evaluation plan as SoA tables
// ---------------------------------------------------------------------------------------------
// Each term i of the merged support (polynomial-major, f's terms first, then start-system terms
// absent from f; reference evaldiff.cpp:189-239) is described by
//   term_info[i] = {poly, k, pos_off, (base_off << 8) | n_base}
//   pos[pos_off + j]   = var | (exponent << 16)   for the k occurring variables, ascending
//   base[base_off + b] = var | ((exponent - 1) << 16) for the variables with exponent >= 2
// i.e. the monomial is (common derivative factor prod x^(e-1)) * (product of the k variables),
// the decomposition of reference polysys.cpp:361-371 / evaldiff.cpp:119-168.
// Coefficients c_start = gamma * c_g and c_target = c_f are stored per term as 2L limbs each.
struct Plan {
  int prec = 0;
  uint32_t L = 1;
  uint32_t dim = 0, n_polys = 0, mon_rows = 0, max_k = 0;
  std::vector<int32_t> term_info;  // 4 per term
  std::vector<uint32_t> pos;
  std::vector<uint32_t> base;
  std::vector<double> coeff;  // per term: c_start (2L) then c_target (2L)
  uint64_t posprod_muls = 0;  // sum of max(0, 3k-5) (+ k-1 for k = 2 ... ) per the schedule
  uint64_t mon_steps = 0;     // reference MonStep count (for documentation / cross-checks)
  uint64_t cmul_steps = 0;    // complex multiplications in the monomial stage
  uint64_t jac_terms = 0;     // Jacobian contributions (sum of k)
  uint64_t jac_scaled = 0;    // contributions with exponent != 1
  // warp-cooperative evaluation: term_slot[i] = first contribution slot of term i (n_terms + 1
  // entries); accumulator a (H_p at a = p, dH_p/dx_v at a = n_polys + p*dim + v) sums the slots
  // acc_idx[acc_off[a] .. acc_off[a+1]) in that order
  std::vector<uint32_t> term_slot, acc_off, acc_idx;
  uint32_t n_terms() const { return static_cast<uint32_t>(term_info.size() / 4); }
  uint32_t n_slots() const { return term_slot.empty() ? 0 : term_slot.back(); }
};

// build_plan<R>(f, g, gamma) with gamma given as 2L limbs at the plan's level
Plan build_plan(const System& f, const System* g, int prec, const double* gamma);

// ---------------------------------------------------------------------------------------------
// start data (homotopy.hpp:31-49)
// ---------------------------------------------------------------------------------------------
struct Starts {
  int prec = 0;
  uint32_t L = 1;
  uint32_t dim = 0;
  bool total_degree = true;
  uint64_t count = 0;
  std::vector<uint32_t> degrees;   // total-degree mode
  std::vector<uint32_t> root_off;  // offset of variable i's root table (in roots, complex units)
  std::vector<double> roots;       // concatenated root tables, 2L limbs per root
  std::vector<double> explicit_x;  // file mode: count * dim * 2L
  void solution(uint64_t index, double* x) const;
};

// total_degree_start<R> (homotopy.cpp:87-113)
std::pair<System, Starts> total_degree_start(const System& f, int prec);

}  // namespace pp
