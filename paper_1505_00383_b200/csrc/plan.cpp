// plan.cpp -- host preprocessor: merged support of target f and start g, per-term monomial
// decomposition, and SoA instruction/coefficient tables for the device.
//
// Term order, coefficient folding and narrowing follow reference evaldiff.cpp:189-239
// (build_plan_impl): per polynomial, f's terms in source order, then g's monomials absent from f;
// c_target = narrow(c_f), c_start = gamma * narrow(c_g) at the run level.  The monomial
// decomposition is (prod over e>=2 of x^(e-1)) * (x_{p0} ... x_{p(k-1)}); the device evaluates the
// product part with the Speelpenning prefix/suffix schedule (3k-5 multiplications) and the common
// factor by square-and-multiply, the exact schedule of evaldiff.cpp:90-161.  The counters below
// reproduce that schedule's step/multiplication counts for documentation and roofline arithmetic.

#include <map>

#include "host.hpp"

namespace pp {

namespace {

template <class R>
cx<R> narrow(const cqd& z) {
  return cx<R>{narrow_qd<R>(z.re), narrow_qd<R>(z.im)};
}

template <class R>
void put(const cx<R>& z, double* out) {
  constexpr int L = level<R>::L;
  for (int l = 0; l < L; ++l) {
    out[l] = level<R>::get(z.re, l);
    out[L + l] = level<R>::get(z.im, l);
  }
}

template <class R>
cx<R> get(const double* in) {
  constexpr int L = level<R>::L;
  cx<R> z;
  for (int l = 0; l < L; ++l) {
    level<R>::set(z.re, l, in[l]);
    level<R>::set(z.im, l, in[L + l]);
  }
  return z;
}

// step / multiplication counts of the reference schedule for one term
void count_schedule(uint32_t k, const std::vector<std::pair<uint32_t, uint32_t>>& base, Plan& p) {
  uint64_t steps = 0, muls = 0;
  if (k == 1) {
    steps += 2;
  } else if (k >= 2) {
    steps += 3ull * k - 2;
    muls += 3ull * k - 5;
    p.posprod_muls += 3ull * k - 5;
  }
  if (!base.empty()) {
    bool init = false;
    for (const auto& [v, e] : base) {
      (void)v;
      if (e == 1) {
        ++steps;
        if (init) ++muls;
        init = true;
        continue;
      }
      ++steps;  // copy into the square-and-multiply accumulator
      for (uint32_t bits = e; bits != 0;) {
        if (bits & 1u) {
          ++steps;
          if (init) ++muls;
          init = true;
        }
        bits >>= 1;
        if (bits != 0) {
          ++steps;
          ++muls;
        }
      }
    }
    steps += k + 1;
    muls += k + 1;
  }
  p.mon_steps += steps;
  p.cmul_steps += muls;
}

template <class R>
void fill_plan(const System& f, const System* g, const double* gamma_limbs, Plan& plan) {
  const cx<R> gamma = get<R>(gamma_limbs);
  constexpr int L = level<R>::L;
  uint32_t row = 0;
  for (uint32_t p = 0; p < plan.n_polys; ++p) {
    std::map<Monomial, size_t> where;
    std::vector<std::pair<Monomial, std::pair<cqd, cqd>>> merged;  // (c_f, c_g)
    const cqd zero{qd_make(0.0), qd_make(0.0)};
    for (const Term& t : f.polys[p]) {
      where[t.mono] = merged.size();
      merged.push_back({t.mono, {t.coeff, zero}});
    }
    if (g != nullptr) {
      for (const Term& t : g->polys[p]) {
        auto it = where.find(t.mono);
        if (it == where.end()) {
          where[t.mono] = merged.size();
          merged.push_back({t.mono, {zero, t.coeff}});
        } else {
          auto& cg = merged[it->second].second.second;
          cg = cadd(cg, t.coeff);
        }
      }
    }
    for (const auto& [mono, cf] : merged) {
      const uint32_t k = static_cast<uint32_t>(mono.factors.size());
      std::vector<std::pair<uint32_t, uint32_t>> base;
      const uint32_t pos_off = static_cast<uint32_t>(plan.pos.size());
      const uint32_t base_off = static_cast<uint32_t>(plan.base.size());
      for (const auto& [v, e] : mono.factors) {
        if (v > 0xffffu || e > 0xffffu) throw InvalidArgument("build_plan: variable index or exponent too large");
        plan.pos.push_back(v | (e << 16));
        if (e > 1) {
          base.emplace_back(v, e - 1);
          plan.base.push_back(v | ((e - 1) << 16));
          ++plan.jac_scaled;
        }
      }
      if (base.size() > 255) throw InvalidArgument("build_plan: too many repeated variables in a monomial");
      plan.term_info.push_back(static_cast<int32_t>(p));
      plan.term_info.push_back(static_cast<int32_t>(k));
      plan.term_info.push_back(static_cast<int32_t>(pos_off));
      plan.term_info.push_back(static_cast<int32_t>((base_off << 8) | static_cast<uint32_t>(base.size())));
      plan.max_k = std::max(plan.max_k, k);
      plan.jac_terms += k;
      row += 1 + k;
      count_schedule(k, base, plan);

      const cx<R> ct = narrow<R>(cf.first);
      const cx<R> cs = cmul(gamma, narrow<R>(cf.second));
      const size_t at = plan.coeff.size();
      plan.coeff.resize(at + 4 * L);
      put(cs, plan.coeff.data() + at);
      put(ct, plan.coeff.data() + at + 2 * L);
    }
  }
  plan.mon_rows = row;
}

// Tables of the warp-cooperative evaluation (one warp per path): every term's products are
// computed independently and parked in contribution slots (slot 0: the term's share of H_poly,
// slots 1..k: its share of dH_poly/dx_var for its k variables in position order); each
// accumulator (H_p, then dH_p/dx_v at np + p*n + v) then sums its slots in plan order, which is
// the reference's sum-stage order (evaldiff.cpp:341-373).
void build_accumulation_lists(Plan& plan) {
  const uint32_t nt = plan.n_terms(), np = plan.n_polys, n = plan.dim;
  plan.term_slot.assign(nt + 1, 0);
  for (uint32_t i = 0; i < nt; ++i) plan.term_slot[i + 1] = plan.term_slot[i] + 1 + plan.term_info[4 * i + 1];
  const uint32_t n_acc = np + np * n;
  std::vector<std::vector<uint32_t>> lists(n_acc);
  for (uint32_t i = 0; i < nt; ++i) {
    const uint32_t p = plan.term_info[4 * i], k = plan.term_info[4 * i + 1], po = plan.term_info[4 * i + 2];
    lists[p].push_back(plan.term_slot[i]);
    for (uint32_t j = 0; j < k; ++j) lists[np + p * n + (plan.pos[po + j] & 0xffffu)].push_back(plan.term_slot[i] + 1 + j);
  }
  plan.acc_off.assign(1, 0);
  plan.acc_idx.clear();
  for (const auto& l : lists) {
    plan.acc_idx.insert(plan.acc_idx.end(), l.begin(), l.end());
    plan.acc_off.push_back(static_cast<uint32_t>(plan.acc_idx.size()));
  }
}

}  // namespace

Plan build_plan(const System& f, const System* g, int prec, const double* gamma) {
  if (g != nullptr && (f.dim != g->dim || f.polys.size() != g->polys.size()))
    throw InvalidArgument("build_plan: dimension mismatch between target and start");
  Plan plan;
  plan.prec = prec;
  plan.dim = f.dim;
  plan.n_polys = static_cast<uint32_t>(f.polys.size());
  switch (prec) {
    case 0:
      plan.L = 1;
      fill_plan<double>(f, g, gamma, plan);
      break;
    case 1:
      plan.L = 2;
      fill_plan<dd_t>(f, g, gamma, plan);
      break;
    case 2:
      plan.L = 4;
      fill_plan<qd_t>(f, g, gamma, plan);
      break;
    default:
      throw InvalidArgument("build_plan: bad precision");
  }
  build_accumulation_lists(plan);
  return plan;
}

}  // namespace pp
