// Test-infrastructure harness around the UNMODIFIED reference library (polypath, built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It exposes the reference's
// own entry points through plain C functions so that tests/, __graft_entry__.smoke() and
// bench.py's reference arm can call them by ctypes.  Nothing in the product links this.
//
// Every function forwards to the reference API named in its comment; no algorithm lives here.

#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>

#include "polypath/homotopy.hpp"
#include "polypath/linalg.hpp"
#include "polypath/parallel.hpp"
#include "polypath/polysys.hpp"
#include "polypath/tracker.hpp"
#include "polypath/xprec_io.hpp"
#include "pp200.h"

using namespace polypath;

namespace {

thread_local std::string g_err;

template <class R>
constexpr int limbs_of() {
  return precision_traits<R>::limbs;
}

template <class R>
void put_real(const R& v, double* out) {
  for (int l = 0; l < limbs_of<R>(); ++l) out[l] = get_limb(v, l);
}

template <class R>
R get_real(const double* in) {
  R v{};
  for (int l = 0; l < limbs_of<R>(); ++l) set_limb(v, l, in[l]);
  return v;
}

template <class R>
void put_cplx(const Cplx<R>& z, double* out) {
  put_real(z.re, out);
  put_real(z.im, out + limbs_of<R>());
}

template <class R>
Cplx<R> get_cplx(const double* in) {
  return {get_real<R>(in), get_real<R>(in + limbs_of<R>())};
}

TrackConfig to_cfg(const pp_track_config* c) {
  TrackConfig t;
  t.residual_tol = c->residual_tol;
  t.update_tol = c->update_tol;
  t.max_newton = c->max_newton;
  t.h_init = c->h_init;
  t.h_min = c->h_min;
  t.h_max = c->h_max;
  t.expand = c->expand;
  t.expand_after = c->expand_after;
  t.contract = c->contract;
  t.divergence_bound = c->divergence_bound;
  t.max_steps = c->max_steps;
  t.batch = c->batch;
  t.workers = c->workers == 0 ? default_worker_count() : c->workers;
  return t;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const ParseError& e) {
    g_err = e.what();
    return PP_E_PARSE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return PP_E_INVALID;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return PP_E_DOMAIN;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PP_E_INVALID;
  }
}

template <class R>
int track_impl(const char* f_text, const char* g_text, const char* starts_text, const double* gamma,
               const pp_track_config* c, uint64_t lo, uint64_t hi, pp_records* out,
               double* wall_ms, uint64_t* rounds, ProgressSink* sink = nullptr) {
  PolySystem f = parse_system(f_text);
  PolySystem g;
  StartData<R> sd;
  if (g_text == nullptr) {
    auto [g0, s0] = total_degree_start<R>(f);
    g = std::move(g0);
    sd = std::move(s0);
  } else {
    g = parse_system(g_text);
    auto cand = parse_solutions(starts_text, g.dim);
    sd = load_start_data<R>(g, cand).data;
  }
  auto h = make_homotopy<R>(f, g, Cplx<R>{R{gamma[0]}, R{gamma[1]}});
  TrackConfig cfg = to_cfg(c);
  auto t0 = std::chrono::steady_clock::now();
  SolutionSet<R> sol = track_all<R>(h, sd, cfg, sink, lo, hi);
  double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (wall_ms) *wall_ms = ms;
  if (rounds) *rounds = sol.total_rounds;
  if (sol.paths.size() > out->capacity) return PP_E_CAPACITY;
  const uint32_t dim = f.dim;
  const int L = limbs_of<R>();
  for (size_t i = 0; i < sol.paths.size(); ++i) {
    const auto& r = sol.paths[i];
    out->path_id[i] = r.path_id;
    out->status[i] = static_cast<int8_t>(r.status);
    out->reason[i] = static_cast<uint8_t>(r.reason);
    out->steps[i] = r.stats.steps;
    out->newton_iters[i] = r.stats.newton_iters;
    out->rejections[i] = r.stats.rejections;
    for (uint32_t v = 0; v < dim; ++v) put_cplx(r.x[v], out->x + (i * dim + v) * 2 * L);
    put_real(r.residual, out->residual + i * L);
  }
  out->count = sol.paths.size();
  return PP_OK;
}

template <class R>
int eval_impl(const char* f_text, const char* g_text, const double* gamma, uint32_t batch,
              const double* points, const double* t, double* sys, double* jac) {
  PolySystem f = parse_system(f_text);
  PolySystem g = g_text ? parse_system(g_text) : total_degree_start<R>(f).first;
  auto h = make_homotopy<R>(f, g, Cplx<R>{get_real<R>(gamma), get_real<R>(gamma + limbs_of<R>())});
  const auto& plan = h.plan;
  BatchWorkspace<R> ws(plan, batch);
  const int L = limbs_of<R>();
  for (uint32_t p = 0; p < batch; ++p) {
    for (uint32_t v = 0; v < plan.dim; ++v)
      ws.points.store(v, p, get_cplx<R>(points + (static_cast<size_t>(p) * plan.dim + v) * 2 * L));
    ws.set_t(p, get_real<R>(t + static_cast<size_t>(p) * L));
  }
  eval_system_batch(plan, ws, 1, nullptr);
  for (uint32_t p = 0; p < batch; ++p) {
    for (uint32_t i = 0; i < plan.n_polys; ++i)
      put_cplx(ws.sys.load(i, p), sys + (static_cast<size_t>(p) * plan.n_polys + i) * 2 * L);
    if (jac)
      for (uint32_t r = 0; r < plan.n_polys * plan.dim; ++r)
        put_cplx(ws.jac.load(r, p),
                 jac + (static_cast<size_t>(p) * plan.n_polys * plan.dim + r) * 2 * L);
  }
  return PP_OK;
}

template <class R>
int lsq_impl(uint32_t n, uint32_t batch, const double* a, const double* b, double* x, uint8_t* ok) {
  const int L = limbs_of<R>();
  for (uint32_t p = 0; p < batch; ++p) {
    DenseMatrix<R> m(n, n);
    std::vector<Cplx<R>> rhs(n), sol(n);
    const double* ap = a + static_cast<size_t>(p) * n * n * 2 * L;
    for (uint32_t j = 0; j < n; ++j)
      for (uint32_t i = 0; i < n; ++i) m.at(i, j) = get_cplx<R>(ap + (j * n + i) * 2 * L);
    for (uint32_t i = 0; i < n; ++i) rhs[i] = get_cplx<R>(b + (static_cast<size_t>(p) * n + i) * 2 * L);
    bool good = least_squares_solve<R>(m, rhs, sol);
    ok[p] = good ? 1 : 0;
    for (uint32_t i = 0; i < n; ++i)
      put_cplx(good ? sol[i] : Cplx<R>{}, x + (static_cast<size_t>(p) * n + i) * 2 * L);
  }
  return PP_OK;
}

template <class R>
int solution_impl(const char* f_text, uint64_t idx, double* x) {
  PolySystem f = parse_system(f_text);
  auto sd = total_degree_start<R>(f).second;
  auto sol = sd.solution(idx);
  for (uint32_t v = 0; v < f.dim; ++v) put_cplx(sol[v], x + v * 2 * limbs_of<R>());
  return PP_OK;
}

// op codes for ref_arith: 0 add, 1 sub, 2 mul, 3 mul by double (b[0]), 4 div, 5 sqrt,
// 6 compare (out[0] = -1/0/1), 7 to_double, 8 complex mul, 9 complex div, 10 cabs,
// 11 R * double via Cplx<R>*double on the real part only (same as 3), 12 pow10_r(b[0])
template <class R>
int arith_impl(int op, const double* a, const double* b, double* out) {
  const int L = limbs_of<R>();
  R x = get_real<R>(a), y = get_real<R>(b);
  switch (op) {
    case 0: put_real<R>(x + y, out); break;
    case 1: put_real<R>(x - y, out); break;
    case 2: put_real<R>(x * y, out); break;
    case 3: {
      if constexpr (std::is_same_v<R, double>) put_real<R>(x * b[0], out);
      else put_real<R>(x * b[0], out);
      break;
    }
    case 4: put_real<R>(x / y, out); break;
    case 5: {
      using polypath::sqrt;
      using std::sqrt;
      put_real<R>(sqrt(x), out);
      break;
    }
    case 6: out[0] = compare(x, y); break;
    case 7: out[0] = to_double(x); break;
    case 8: put_cplx<R>(get_cplx<R>(a) * get_cplx<R>(b), out); break;
    case 9: put_cplx<R>(get_cplx<R>(a) / get_cplx<R>(b), out); break;
    case 10: put_real<R>(cabs(get_cplx<R>(a)), out); break;
    case 12: put_real<R>(pow10_r<R>(static_cast<long>(b[0])), out); break;
    default: return PP_E_INVALID;
  }
  (void)L;
  return PP_OK;
}

template <class R>
int parse_impl(const char* s, double* out) {
  R v{};
  if (!parse_decimal(s, v)) return PP_E_PARSE;
  put_real(v, out);
  return PP_OK;
}

template <class R>
int print_impl(const double* in, char* buf, size_t cap) {
  std::string s = to_decimal(get_real<R>(in));
  if (s.size() + 1 > cap) return PP_E_CAPACITY;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return PP_OK;
}

template <class R>
int plan_impl(const char* f_text, const char* g_text, uint32_t* info, double* coeffs) {
  PolySystem f = parse_system(f_text);
  PolySystem g = g_text ? parse_system(g_text) : total_degree_start<R>(f).first;
  auto h = make_homotopy<R>(f, g, Cplx<R>{R{1.0}, R{}});
  const auto& plan = h.plan;
  uint32_t steps = 0, jac = 0, maxk = 0;
  for (const auto& t : plan.terms) {
    steps += static_cast<uint32_t>(t.steps.size());
    jac += static_cast<uint32_t>(t.positions.size());
    maxk = std::max<uint32_t>(maxk, static_cast<uint32_t>(t.positions.size()));
  }
  info[0] = plan.dim;
  info[1] = plan.n_polys;
  info[2] = static_cast<uint32_t>(plan.terms.size());
  info[3] = plan.mon_rows;
  info[4] = steps;
  info[5] = static_cast<uint32_t>(plan.total_posprod_muls());
  info[6] = jac;
  info[7] = maxk;
  if (coeffs) {
    const int L = limbs_of<R>();
    for (size_t i = 0; i < plan.terms.size(); ++i) {
      put_cplx(plan.c_start[i], coeffs + (2 * i) * 2 * L);
      put_cplx(plan.c_target[i], coeffs + (2 * i + 1) * 2 * L);
    }
  }
  return PP_OK;
}

// the reference plan's term structure, in the neutral layout the C restatement consumes:
// term_info[4*i] = {poly, k, pos_off, 0}; pos[pos_off + j] = var | (exponent << 16);
// coeff[i] = (c_start, c_target), 2L doubles each
template <class R>
int plan_terms_impl(const char* f_text, const char* g_text, const double* gamma, int32_t* term_info,
                    uint32_t* pos, double* coeff, uint32_t* counts) {
  PolySystem f = parse_system(f_text);
  PolySystem g = g_text ? parse_system(g_text) : total_degree_start<R>(f).first;
  auto h = make_homotopy<R>(f, g, Cplx<R>{get_real<R>(gamma), get_real<R>(gamma + limbs_of<R>())});
  const auto& plan = h.plan;
  const int L = limbs_of<R>();
  uint32_t off = 0;
  for (size_t i = 0; i < plan.terms.size(); ++i) {
    const auto& t = plan.terms[i];
    if (term_info) {
      term_info[4 * i + 0] = static_cast<int32_t>(t.poly);
      term_info[4 * i + 1] = static_cast<int32_t>(t.positions.size());
      term_info[4 * i + 2] = static_cast<int32_t>(off);
      term_info[4 * i + 3] = 0;
    }
    for (size_t j = 0; j < t.positions.size(); ++j) {
      if (pos) pos[off] = t.positions[j] | (t.pos_exponents[j] << 16);
      ++off;
    }
    if (coeff) {
      put_cplx(plan.c_start[i], coeff + (2 * i) * 2 * L);
      put_cplx(plan.c_target[i], coeff + (2 * i + 1) * 2 * L);
    }
  }
  counts[0] = plan.dim;
  counts[1] = plan.n_polys;
  counts[2] = static_cast<uint32_t>(plan.terms.size());
  counts[3] = off;
  return PP_OK;
}

template <class F>
int dispatch(int prec, F&& f) {
  switch (prec) {
    case PP_D: return f(double{});
    case PP_DD: return f(DD{});
    case PP_QD: return f(QD{});
    default: g_err = "bad precision"; return PP_E_INVALID;
  }
}

}  // namespace

// PathBatch::set_prediction + newton_correct (tracker.hpp:135-136, tracker.cpp:216-274) for
// `batch` (t, x) pairs on f with start g and gamma (2L limbs), cohort width = batch
template <class R>
int newton_impl(const char* f_text, const char* g_text, const double* gamma, const pp_track_config* c, uint32_t batch,
                const double* t, double* x, uint32_t* iters, uint8_t* corrected, uint32_t* rounds) {
  PolySystem f = parse_system(f_text);
  PolySystem g = g_text ? parse_system(g_text) : total_degree_start<R>(f).first;
  auto h = make_homotopy<R>(f, g, Cplx<R>{get_real<R>(gamma), get_real<R>(gamma + limbs_of<R>())});
  TrackConfig cfg = to_cfg(c);
  const uint32_t dim = f.dim;
  const int L = limbs_of<R>();
  PathBatch<R> b(h, cfg, batch);
  std::vector<Cplx<R>> xs(dim);
  for (uint32_t i = 0; i < batch; ++i) {
    for (uint32_t v = 0; v < dim; ++v) xs[v] = get_cplx<R>(x + (static_cast<size_t>(i) * dim + v) * 2 * L);
    b.seed(i, xs);
  }
  for (uint32_t i = 0; i < batch; ++i) {
    for (uint32_t v = 0; v < dim; ++v) xs[v] = get_cplx<R>(x + (static_cast<size_t>(i) * dim + v) * 2 * L);
    b.set_prediction(i, get_real<R>(t + static_cast<size_t>(i) * L), xs);
  }
  *rounds = b.newton_correct();
  for (uint32_t i = 0; i < batch; ++i) {
    iters[i] = b.last_iterations(i);
    corrected[i] = b.last_corrected(i) ? 1 : 0;
    auto w = b.working_point(i);
    for (uint32_t v = 0; v < dim; ++v) put_cplx(w[v], x + (static_cast<size_t>(i) * dim + v) * 2 * L);
  }
  return PP_OK;
}

extern "C" {

int ref_newton(const char* f_text, const char* g_text, int prec, const double* gamma, const pp_track_config* cfg,
               uint32_t batch, const double* t, double* x, uint32_t* iters, uint8_t* corrected, uint32_t* rounds) {
  return guarded([&] {
    return dispatch(prec, [&](auto tag) {
      using R = decltype(tag);
      return newton_impl<R>(f_text, g_text, gamma, cfg, batch, t, x, iters, corrected, rounds);
    });
  });
}

const char* ref_last_error(void) { return g_err.c_str(); }

unsigned ref_default_workers(void) { return default_worker_count(); }

void ref_random_gamma(uint64_t seed, double* re, double* im) {
  Cplx<double> g = random_gamma(seed);
  *re = g.re;
  *im = g.im;
}

void ref_track_config_defaults(int prec, pp_track_config* c) {
  TrackConfig t = TrackConfig::defaults(static_cast<Precision>(prec));
  std::memset(c, 0, sizeof *c);
  c->residual_tol = t.residual_tol;
  c->update_tol = t.update_tol;
  c->max_newton = t.max_newton;
  c->expand_after = t.expand_after;
  c->h_init = t.h_init;
  c->h_min = t.h_min;
  c->h_max = t.h_max;
  c->expand = t.expand;
  c->contract = t.contract;
  c->divergence_bound = t.divergence_bound;
  c->max_steps = t.max_steps;
  c->batch = t.batch;
  c->workers = t.workers;
}

// track_all<R> (tracker.cpp:511-540).  g_text == NULL: total-degree start (homotopy.cpp:87-113);
// else g_text + starts_text through parse_solutions/load_start_data.  gamma = (re, im) doubles.
int ref_track(const char* f_text, const char* g_text, const char* starts_text, int prec,
              const double* gamma, const pp_track_config* cfg, uint64_t lo, uint64_t hi,
              pp_records* out, double* wall_ms, uint64_t* rounds) {
  return guarded([&] {
    return dispatch(prec, [&](auto tag) {
      using R = decltype(tag);
      return track_impl<R>(f_text, g_text, starts_text, gamma, cfg, lo, hi, out, wall_ms, rounds);
    });
  });
}

// track_all<R> with a ProgressSink (tracker.hpp:62-70) that records every StepEvent in emission
// order (tracker.cpp:312-315); *n_ev = events emitted (up to ev_cap are stored)
int ref_track_events(const char* f_text, const char* g_text, const char* starts_text, int prec,
                     const double* gamma, const pp_track_config* cfg, uint64_t lo, uint64_t hi,
                     pp_records* out, pp_step_event* ev, uint64_t ev_cap, uint64_t* n_ev) {
  uint64_t k = 0;
  ProgressSink sink = [&](const StepEvent& e) {
    if (k < ev_cap) {
      pp_step_event& o = ev[k];
      std::memset(&o, 0, sizeof o);
      o.path_id = e.path_id;
      o.t = e.t;
      o.h = e.h;
      o.newton_iters = e.newton_iters;
      o.status = e.status;
      o.accepted = e.accepted ? 1 : 0;
    }
    ++k;
  };
  int rc = guarded([&] {
    return dispatch(prec, [&](auto tag) {
      using R = decltype(tag);
      return track_impl<R>(f_text, g_text, starts_text, gamma, cfg, lo, hi, out, nullptr, nullptr, &sink);
    });
  });
  *n_ev = k;
  return rc;
}

// eval_system_batch (evaldiff.cpp:473-488); gamma given as 2L limbs
int ref_eval(const char* f_text, const char* g_text, int prec, const double* gamma, uint32_t batch,
             const double* points, const double* t, double* sys, double* jac) {
  return guarded([&] {
    return dispatch(prec, [&](auto tag) {
      using R = decltype(tag);
      return eval_impl<R>(f_text, g_text, gamma, batch, points, t, sys, jac);
    });
  });
}

// least_squares_solve (linalg.hpp:110-125)
int ref_lsq(int prec, uint32_t n, uint32_t batch, const double* a, const double* b, double* x,
            uint8_t* ok) {
  return guarded([&] {
    return dispatch(prec, [&](auto tag) {
      using R = decltype(tag);
      return lsq_impl<R>(n, batch, a, b, x, ok);
    });
  });
}

// StartData::solution (homotopy.cpp:73-85) of the total-degree start of f
int ref_td_solution(const char* f_text, int prec, uint64_t idx, double* x) {
  return guarded([&] {
    return dispatch(prec, [&](auto tag) {
      using R = decltype(tag);
      return solution_impl<R>(f_text, idx, x);
    });
  });
}

int ref_arith(int prec, int op, const double* a, const double* b, double* out) {
  return guarded([&] {
    return dispatch(prec, [&](auto tag) {
      using R = decltype(tag);
      return arith_impl<R>(op, a, b, out);
    });
  });
}

// parse_decimal (xprec_io.cpp:121-193)
int ref_parse_decimal(int prec, const char* s, double* out) {
  return guarded([&] {
    return dispatch(prec, [&](auto tag) {
      using R = decltype(tag);
      return parse_impl<R>(s, out);
    });
  });
}

// to_decimal (xprec_io.cpp:198-212)
int ref_to_decimal(int prec, const double* in, char* buf, size_t cap) {
  return guarded([&] {
    return dispatch(prec, [&](auto tag) {
      using R = decltype(tag);
      return print_impl<R>(in, buf, cap);
    });
  });
}

// build_plan (evaldiff.cpp:189-246) geometry: info[8] = dim, n_polys, terms, mon_rows, steps,
// posprod_muls, jacobian contributions, max k; coeffs (optional) = per term (c_start, c_target)
int ref_plan_info(const char* f_text, const char* g_text, int prec, uint32_t* info, double* coeffs) {
  return guarded([&] {
    return dispatch(prec, [&](auto tag) {
      using R = decltype(tag);
      return plan_impl<R>(f_text, g_text, info, coeffs);
    });
  });
}

// build_plan term structure and coefficients (evaldiff.cpp:189-239); call once with NULL arrays
// to size them (counts = dim, n_polys, terms, positions)
int ref_plan_terms(const char* f_text, const char* g_text, int prec, const double* gamma, int32_t* term_info,
                   uint32_t* pos, double* coeff, uint32_t* counts) {
  return guarded([&] {
    return dispatch(prec, [&](auto tag) {
      using R = decltype(tag);
      return plan_terms_impl<R>(f_text, g_text, gamma, term_info, pos, coeff, counts);
    });
  });
}

// print_system(parse_system(text)) (polysys.cpp:273-313)
int ref_print_system(const char* text, char* buf, size_t cap) {
  return guarded([&] {
    std::string s = print_system(parse_system(text));
    if (s.size() + 1 > cap) return PP_E_CAPACITY;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return PP_OK;
  });
}

// cyclic_system(n) printed (polysys.cpp:315-336)
int ref_cyclic_text(uint32_t n, char* buf, size_t cap) {
  return guarded([&] {
    std::string s = print_system(cyclic_system(n));
    if (s.size() + 1 > cap) return PP_E_CAPACITY;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return PP_OK;
  });
}

}  // extern "C"
