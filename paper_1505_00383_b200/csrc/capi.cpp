// capi.cpp -- the extern "C" boundary declared in include/pp200.h.
//
// Each entry point maps one reference call (cited in pp200.h) onto the host model (host.hpp) and
// the CUDA path (device.hpp), and maps C++ exceptions onto error codes exactly where the
// reference throws: InvalidArgument -> PP_E_INVALID (std::invalid_argument), ParseFailure ->
// PP_E_PARSE (polypath::ParseError), CudaFailure -> PP_E_CUDA.

#include <algorithm>
#include <charconv>
#include <cstring>
#include <map>
#include <vector>
#include <memory>
#include <mutex>
#include <string>

#include "device.hpp"
#include "json_number.hpp"
#include "host.hpp"
#include "pp200.h"

struct pp_system {
  pp::System sys;
};

struct pp_starts {
  pp::Starts st;
};

struct pp_homotopy {
  pp::System f, g;
  pp::Plan plan;
  std::mutex mu;
  std::map<int, pp::DevicePlan*> uploaded;  // device -> resident plan tables
  ~pp_homotopy() {
    for (auto& [d, p] : uploaded) pp::device_plan_free(p);
  }
  pp::DevicePlan* on(int device) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = uploaded.find(device);
    if (it != uploaded.end()) return it->second;
    pp::DevicePlan* p = pp::device_plan_upload(plan, device);
    uploaded[device] = p;
    return p;
  }
};

namespace {

thread_local std::string g_error;

int limbs_of(int prec) { return prec == PP_D ? 1 : prec == PP_DD ? 2 : prec == PP_QD ? 4 : 0; }

template <class F>
int guard(F&& f) {
  try {
    g_error.clear();
    return f();
  } catch (const pp::ParseFailure& e) {
    g_error = std::string(e.what()) + " at line " + std::to_string(e.line) + ", column " + std::to_string(e.col);
    return PP_E_PARSE;
  } catch (const pp::CudaFailure& e) {
    g_error = e.what();
    return PP_E_CUDA;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return PP_E_INVALID;
  } catch (const std::bad_alloc&) {
    g_error = "out of memory";
    return PP_E_NOMEM;
  } catch (const std::exception& e) {
    g_error = e.what();
    return PP_E_INVALID;
  }
}

void need(bool cond, const char* msg) {
  if (!cond) throw pp::InvalidArgument(msg);
}

}  // namespace

extern "C" {

const char* pp_version(void) { return "pp200 0.2 (sm_100a)"; }

int pp_device_count(void) { return pp::device_count(); }

int pp_device_init(int device) {
  int rc = guard([&] {
    pp::device_init(device);
    return PP_OK;
  });
  if (rc != PP_OK) return rc;
  // one tiny tracking run (x^2 - 4 from x^2 - 1, two paths in complex double), so that the first
  // real call does not pay for the first use of the stream-ordered allocator, graph capture and
  // instantiation, or the first launches either
  const char f_text[] = "1; x0^2 - 4;", g_text[] = "1; x0^2 - 1;";
  pp_system *f = nullptr, *g = nullptr;
  pp_homotopy* h = nullptr;
  pp_starts* st = nullptr;
  const double gam[2] = {1.0, 0.0}, x0[4] = {1.0, 0.0, -1.0, 0.0};
  uint64_t id[2];
  int8_t status[2];
  uint8_t reason[2];
  uint32_t steps[2], newton[2], rej[2];
  double x[4], res[2];
  pp_records rec{2, 0, id, status, reason, steps, newton, rej, x, res};
  pp_track_config c;
  pp_track_config_defaults(PP_D, &c);
  rc = pp_system_parse(f_text, sizeof f_text - 1, &f);
  if (rc == PP_OK) rc = pp_system_parse(g_text, sizeof g_text - 1, &g);
  if (rc == PP_OK) rc = pp_make_homotopy(f, g, PP_D, gam, &h);
  if (rc == PP_OK) rc = pp_starts_explicit(PP_D, 1, 2, x0, &st);
  if (rc == PP_OK) rc = pp_track_all(h, st, &c, 0, 2, device, &rec, nullptr);
  pp_starts_free(st);
  pp_homotopy_free(h);
  pp_system_free(g);
  pp_system_free(f);
  return rc;
}
const char* pp_last_error(void) { return g_error.c_str(); }
int pp_limbs(int prec) { return limbs_of(prec); }

int pp_system_parse(const char* text, size_t len, pp_system** out) {
  return guard([&] {
    need(text != nullptr && out != nullptr, "pp_system_parse: null argument");
    auto s = std::make_unique<pp_system>();
    s->sys = pp::parse_system(std::string_view(text, len));
    *out = s.release();
    return PP_OK;
  });
}

int pp_system_from_terms(uint32_t dim, uint32_t n_polys, const uint32_t* term_count, const uint32_t* n_factors,
                         const uint32_t* factors, const double* coeff, pp_system** out) {
  return guard([&] {
    need(out != nullptr && (n_polys == 0 || term_count != nullptr), "pp_system_from_terms: null argument");
    need(n_polys > 0, "system has no polynomials");
    auto s = std::make_unique<pp_system>();
    s->sys.dim = dim;
    s->sys.polys.resize(n_polys);
    size_t t = 0, f = 0;
    for (uint32_t p = 0; p < n_polys; ++p) {
      for (uint32_t i = 0; i < term_count[p]; ++i, ++t) {
        pp::Term term;
        const double* c = coeff + t * 8;
        term.coeff = pp::cqd{pp::qd_t{c[0], c[1], c[2], c[3]}, pp::qd_t{c[4], c[5], c[6], c[7]}};
        for (uint32_t k = 0; k < n_factors[t]; ++k, ++f) {
          const uint32_t var = factors[2 * f], e = factors[2 * f + 1];
          need(var < dim && e >= 1, "pp_system_from_terms: bad factor");
          need(term.mono.factors.empty() || term.mono.factors.back().first < var,
               "pp_system_from_terms: factors must be sorted by variable");
          term.mono.factors.emplace_back(var, e);
        }
        s->sys.polys[p].push_back(std::move(term));
      }
    }
    s->sys.refresh_degrees();
    *out = s.release();
    return PP_OK;
  });
}

int pp_system_cyclic(uint32_t n, pp_system** out) {
  return guard([&] {
    need(out != nullptr, "pp_system_cyclic: null argument");
    auto s = std::make_unique<pp_system>();
    s->sys = pp::cyclic_system(n);
    *out = s.release();
    return PP_OK;
  });
}

int pp_system_print(const pp_system* s, char* buf, size_t cap, size_t* needed) {
  return guard([&] {
    need(s != nullptr, "pp_system_print: null system");
    std::string text = pp::print_system(s->sys);
    if (needed) *needed = text.size() + 1;
    if (buf == nullptr || cap < text.size() + 1) return PP_E_CAPACITY;
    std::memcpy(buf, text.c_str(), text.size() + 1);
    return PP_OK;
  });
}

int pp_system_stats(const pp_system* s, uint32_t* dim, uint32_t* n_polys, uint64_t* n_monomials,
                    uint64_t* total_degree, int* overflow) {
  return guard([&] {
    need(s != nullptr, "pp_system_stats: null system");
    if (dim) *dim = s->sys.dim;
    if (n_polys) *n_polys = static_cast<uint32_t>(s->sys.polys.size());
    if (n_monomials) *n_monomials = s->sys.monomial_count();
    uint64_t td = 1;
    int of = 0;
    for (uint32_t d : s->sys.degrees) {
      if (__builtin_mul_overflow(td, static_cast<uint64_t>(d), &td)) {
        td = UINT64_MAX;
        of = 1;
        break;
      }
    }
    if (total_degree) *total_degree = td;
    if (overflow) *overflow = of;
    return PP_OK;
  });
}

int pp_system_degrees(const pp_system* s, uint32_t* degrees) {
  return guard([&] {
    need(s != nullptr && degrees != nullptr, "pp_system_degrees: null argument");
    std::copy(s->sys.degrees.begin(), s->sys.degrees.end(), degrees);
    return PP_OK;
  });
}

void pp_system_free(pp_system* s) { delete s; }

void pp_random_gamma(uint64_t seed, double* re, double* im) { pp::random_gamma(seed, *re, *im); }

int pp_total_degree_start(const pp_system* f, int prec, pp_system** g_out, pp_starts** out) {
  return guard([&] {
    need(f != nullptr && out != nullptr, "pp_total_degree_start: null argument");
    need(limbs_of(prec) > 0, "pp_total_degree_start: bad precision");
    auto [g, st] = pp::total_degree_start(f->sys, prec);
    auto so = std::make_unique<pp_starts>();
    so->st = std::move(st);
    if (g_out) {
      auto go = std::make_unique<pp_system>();
      go->sys = std::move(g);
      *g_out = go.release();
    }
    *out = so.release();
    return PP_OK;
  });
}

int pp_starts_explicit(int prec, uint32_t dim, uint64_t count, const double* x, pp_starts** out) {
  return guard([&] {
    const int L = limbs_of(prec);
    need(L > 0 && out != nullptr && (x != nullptr || count == 0), "pp_starts_explicit: bad argument");
    auto so = std::make_unique<pp_starts>();
    so->st.prec = prec;
    so->st.L = L;
    so->st.dim = dim;
    so->st.total_degree = false;
    so->st.count = count;
    so->st.explicit_x.assign(x, x + count * dim * 2 * L);
    *out = so.release();
    return PP_OK;
  });
}

int pp_starts_roots(int prec, uint32_t dim, const uint32_t* degrees, const double* roots, pp_starts** out) {
  return guard([&] {
    const int L = limbs_of(prec);
    need(L > 0 && out != nullptr && dim > 0 && degrees != nullptr && roots != nullptr,
         "pp_starts_roots: bad argument");
    auto so = std::make_unique<pp_starts>();
    so->st.prec = prec;
    so->st.L = L;
    so->st.dim = dim;
    so->st.total_degree = true;
    uint64_t count = 1, total = 0;
    for (uint32_t i = 0; i < dim; ++i) {
      if (degrees[i] == 0) throw pp::InvalidArgument("pp_starts_roots: zero degree");
      so->st.degrees.push_back(degrees[i]);
      so->st.root_off.push_back(static_cast<uint32_t>(total));
      total += degrees[i];
      count *= degrees[i];  // as total_degree_start (homotopy.cpp:102)
    }
    so->st.count = count;
    so->st.roots.assign(roots, roots + total * 2 * L);
    *out = so.release();
    return PP_OK;
  });
}

int pp_load_start_data(const pp_system* g, int prec, const char* text, size_t len, double start_tol,
                       int device, pp_starts** out, uint64_t* rejected_idx, double* rejected_resid,
                       uint64_t rejected_cap, uint64_t* n_rejected) {
  return guard([&] {
    const int L = limbs_of(prec);
    need(g != nullptr && text != nullptr && out != nullptr && L > 0, "pp_load_start_data: bad argument");
    auto cand = pp::parse_solutions(std::string_view(text, len), g->sys.dim);
    const uint32_t dim = g->sys.dim, w = 2 * L;
    // candidates narrowed to the run level, then H_g(x) evaluated on the device at t = 1 against
    // the plan of g alone (homotopy.cpp:121-131)
    std::vector<double> xs(cand.size() * dim * w), ts(cand.size() * L, 0.0);
    for (size_t i = 0; i < cand.size(); ++i) {
      for (uint32_t v = 0; v < dim; ++v) {
        double* dst = xs.data() + (i * dim + v) * w;
        const pp::cqd& z = cand[i][v];
        switch (prec) {
          case PP_D:
            dst[0] = pp::narrow_qd<double>(z.re);
            dst[1] = pp::narrow_qd<double>(z.im);
            break;
          case PP_DD: {
            pp::dd_t re = pp::narrow_qd<pp::dd_t>(z.re), im = pp::narrow_qd<pp::dd_t>(z.im);
            dst[0] = re.hi, dst[1] = re.lo, dst[2] = im.hi, dst[3] = im.lo;
            break;
          }
          default:
            dst[0] = z.re.c0, dst[1] = z.re.c1, dst[2] = z.re.c2, dst[3] = z.re.c3;
            dst[4] = z.im.c0, dst[5] = z.im.c1, dst[6] = z.im.c2, dst[7] = z.im.c3;
        }
      }
      ts[i * L] = 1.0;
    }
    const double gamma1[8] = {1.0, 0, 0, 0, 0, 0, 0, 0};
    double gl[8] = {0};
    gl[0] = gamma1[0];
    pp::Plan plan = pp::build_plan(g->sys, nullptr, prec, gl);
    const uint32_t np = plan.n_polys;
    std::vector<double> vals(cand.size() * np * w);
    if (!cand.empty()) {
      pp::DevicePlan* dp = pp::device_plan_upload(plan, device);
      try {
        pp::device_eval(plan, dp, static_cast<uint32_t>(cand.size()), xs.data(), ts.data(), vals.data(), nullptr,
                        device);
      } catch (...) {
        pp::device_plan_free(dp);
        throw;
      }
      pp::device_plan_free(dp);
    }
    auto so = std::make_unique<pp_starts>();
    so->st.prec = prec;
    so->st.L = L;
    so->st.dim = dim;
    so->st.total_degree = false;
    uint64_t nrej = 0;
    for (size_t i = 0; i < cand.size(); ++i) {
      // resid = max_i to_double(|v_i|), computed by the device evaluation's own norm primitive
      double resid = 0.0;
      for (uint32_t p = 0; p < np; ++p) {
        const double* v = vals.data() + (i * np + p) * w;
        double m;
        switch (prec) {
          case PP_D: m = pp::cabsd(pp::cx<double>{v[0], v[1]}); break;
          case PP_DD: m = pp::cabsd(pp::cx<pp::dd_t>{{v[0], v[1]}, {v[2], v[3]}}); break;
          default: m = pp::cabsd(pp::cx<pp::qd_t>{{v[0], v[1], v[2], v[3]}, {v[4], v[5], v[6], v[7]}});
        }
        resid = pp::f_max(resid, m);
      }
      if (resid < start_tol) {
        so->st.explicit_x.insert(so->st.explicit_x.end(), xs.begin() + i * dim * w, xs.begin() + (i + 1) * dim * w);
      } else {
        if (nrej < rejected_cap) {
          if (rejected_idx) rejected_idx[nrej] = i;
          if (rejected_resid) rejected_resid[nrej] = resid;
        }
        ++nrej;
      }
    }
    so->st.count = so->st.explicit_x.size() / (static_cast<size_t>(dim) * w);
    if (n_rejected) *n_rejected = nrej;
    *out = so.release();
    return PP_OK;
  });
}

uint64_t pp_starts_count(const pp_starts* s) { return s ? s->st.count : 0; }

int pp_starts_solution(const pp_starts* s, uint64_t index, double* x) {
  return guard([&] {
    need(s != nullptr && x != nullptr, "pp_starts_solution: null argument");
    need(index < s->st.count, "pp_starts_solution: index out of range");
    s->st.solution(index, x);
    return PP_OK;
  });
}

void pp_starts_free(pp_starts* s) { delete s; }

int pp_make_homotopy(const pp_system* f, const pp_system* g, int prec, const double* gamma, pp_homotopy** out) {
  return guard([&] {
    const int L = limbs_of(prec);
    need(f != nullptr && g != nullptr && gamma != nullptr && out != nullptr && L > 0,
         "pp_make_homotopy: bad argument");
    if (f->sys.dim != g->sys.dim || f->sys.polys.size() != g->sys.polys.size())
      throw pp::InvalidArgument("make_homotopy: target and start dimensions differ");
    // |gamma| = 1 within 1e-12, measured as sqrt(to_double(|gamma|^2)) (homotopy.cpp:11-13)
    double mod2;
    switch (prec) {
      case PP_D: mod2 = pp::cabs2(pp::cx<double>{gamma[0], gamma[1]}); break;
      case PP_DD: mod2 = pp::rtod(pp::cabs2(pp::cx<pp::dd_t>{{gamma[0], gamma[1]}, {gamma[2], gamma[3]}})); break;
      default:
        mod2 = pp::rtod(pp::cabs2(pp::cx<pp::qd_t>{{gamma[0], gamma[1], gamma[2], gamma[3]},
                                                  {gamma[4], gamma[5], gamma[6], gamma[7]}}));
    }
    if (std::fabs(std::sqrt(mod2) - 1.0) > 1e-12) throw pp::InvalidArgument("make_homotopy: gamma must have unit modulus");
    auto h = std::make_unique<pp_homotopy>();
    h->plan = pp::build_plan(f->sys, &g->sys, prec, gamma);
    h->f = f->sys;
    h->g = g->sys;
    *out = h.release();
    return PP_OK;
  });
}

int pp_homotopy_info(const pp_homotopy* h, uint32_t* dim, uint32_t* n_polys, uint32_t* n_terms,
                     uint32_t* mon_rows, uint32_t* max_k, uint64_t* posprod_muls) {
  return guard([&] {
    need(h != nullptr, "pp_homotopy_info: null homotopy");
    if (dim) *dim = h->plan.dim;
    if (n_polys) *n_polys = h->plan.n_polys;
    if (n_terms) *n_terms = h->plan.n_terms();
    if (mon_rows) *mon_rows = h->plan.mon_rows;
    if (max_k) *max_k = h->plan.max_k;
    if (posprod_muls) *posprod_muls = h->plan.posprod_muls;
    return PP_OK;
  });
}

// extended plan counters used for roofline arithmetic: [mon_steps, cmul_steps, jac_terms,
// jac_scaled, n_base]
int pp_homotopy_counts(const pp_homotopy* h, uint64_t* counts) {
  return guard([&] {
    need(h != nullptr && counts != nullptr, "pp_homotopy_counts: null argument");
    counts[0] = h->plan.mon_steps;
    counts[1] = h->plan.cmul_steps;
    counts[2] = h->plan.jac_terms;
    counts[3] = h->plan.jac_scaled;
    counts[4] = h->plan.base.size();
    return PP_OK;
  });
}

void pp_homotopy_free(pp_homotopy* h) { delete h; }

void pp_track_config_defaults(int prec, pp_track_config* c) {
  std::memset(c, 0, sizeof *c);
  c->residual_tol = c->update_tol = prec == PP_D ? 1e-8 : (prec == PP_DD ? 1e-14 : 1e-28);
  c->h_min = prec == PP_D ? 1e-6 : 1e-8;
  c->max_newton = 3;
  c->expand_after = 2;
  c->h_init = 0.05;
  c->h_max = 0.1;
  c->expand = 1.5;
  c->contract = 0.5;
  c->divergence_bound = 1e8;
  c->max_steps = 10000;
  c->batch = 64;
  c->workers = 1;
}

int pp_track_config_validate(const pp_track_config* c) {
  return guard([&] {
    need(c != nullptr, "TrackConfig: null");
    if (!(c->h_min > 0.0 && c->h_min <= c->h_init && c->h_init <= c->h_max && c->h_max <= 0.1))
      throw pp::InvalidArgument("TrackConfig: need 0 < h_min <= h_init <= h_max <= 0.1");
    if (c->max_newton < 1) throw pp::InvalidArgument("TrackConfig: max_newton must be >= 1");
    if (c->batch < 1) throw pp::InvalidArgument("TrackConfig: batch must be >= 1");
    if (!(c->expand >= 1.0) || !(c->contract > 0.0 && c->contract < 1.0))
      throw pp::InvalidArgument("TrackConfig: bad expand/contract factors");
    if (!(c->residual_tol > 0.0) || !(c->update_tol > 0.0))
      throw pp::InvalidArgument("TrackConfig: tolerances must be positive");
    return PP_OK;
  });
}

uint64_t pp_shard_size(uint64_t lo, uint64_t hi, const pp_shard* shard) {
  pp::TrackShard sh;
  if (shard != nullptr && shard->count > 1) sh = {shard->index, shard->count, shard->block ? shard->block : 1};
  return pp::shard_size(lo, hi, sh);
}

int pp_track_all_ex(const pp_homotopy* h, const pp_starts* s, const pp_track_config* cfg, uint64_t lo,
                    uint64_t hi, const pp_shard* shard, pp_event_sink sink, void* sink_user, int device,
                    pp_records* out, pp_run_stats* stats) {
  int rc = pp_track_config_validate(cfg);
  if (rc != PP_OK) return rc;
  return guard([&] {
    need(h != nullptr && s != nullptr && out != nullptr, "track_all: null argument");
    if (s->st.count == 0) throw pp::InvalidArgument("track_all: no start solutions");
    need(s->st.prec == h->plan.prec, "track_all: start data and homotopy precision differ");
    need(s->st.dim == h->plan.dim, "track_all: start dimension differs from the homotopy");
    need(h->plan.n_polys == h->plan.dim, "track_all: the homotopy must be square");
    pp::TrackShard sh;
    if (shard != nullptr) {
      need(shard->count >= 1 && shard->index < shard->count && shard->block >= 1, "track_all: bad shard");
      sh = {shard->index, shard->count, shard->block};
    }
    const uint64_t end = std::min<uint64_t>(s->st.count, hi);
    if (stats) std::memset(stats, 0, sizeof *stats);
    out->count = 0;
    if (lo >= end) return PP_OK;
    const uint64_t n = pp::shard_size(lo, end, sh);
    if (n == 0) return PP_OK;
    if (out->capacity < n) return PP_E_CAPACITY;
    pp_homotopy* hm = const_cast<pp_homotopy*>(h);
    pp::device_track(hm->plan, hm->on(device), s->st, *cfg, lo, end, sh, pp::EventSink{sink, sink_user}, device, out,
                     stats);
    return PP_OK;
  });
}

int pp_track_all(const pp_homotopy* h, const pp_starts* s, const pp_track_config* cfg, uint64_t lo,
                 uint64_t hi, int device, pp_records* out, pp_run_stats* stats) {
  return pp_track_all_ex(h, s, cfg, lo, hi, nullptr, nullptr, nullptr, device, out, stats);
}

int pp_eval_batch(const pp_homotopy* h, uint32_t batch, const double* points, const double* t, double* sys,
                  double* jac, int device) {
  return guard([&] {
    need(h != nullptr && (batch == 0 || (points && t && sys)), "pp_eval_batch: null argument");
    pp_homotopy* hm = const_cast<pp_homotopy*>(h);
    pp::device_eval(hm->plan, hm->on(device), batch, points, t, sys, jac, device);
    return PP_OK;
  });
}

int pp_lsq_batch_mn(int prec, uint32_t m, uint32_t n, uint32_t batch, const double* a, const double* b, double* x,
                    uint8_t* ok, double* q, double* r, int device) {
  return guard([&] {
    need(limbs_of(prec) > 0 && n >= 1 && m >= n, "pp_lsq_batch: bad argument (need m >= n >= 1)");
    need(batch == 0 || (a && b && x && ok), "pp_lsq_batch: null argument");
    pp::device_lsq(prec, m, n, batch, a, b, x, ok, q, r, device);
    return PP_OK;
  });
}

int pp_lsq_batch(int prec, uint32_t n, uint32_t batch, const double* a, const double* b, double* x, uint8_t* ok,
                 int device) {
  return pp_lsq_batch_mn(prec, n, n, batch, a, b, x, ok, nullptr, nullptr, device);
}

// ---- output records: the reference CLI's JSON lines (polypath_main.cpp:125-189) ----
}  // extern "C"

namespace {
// a double as nlohmann::json::dump prints it (json_number.cpp)
void put_double(std::string& o, double v) { pp::json_double(o, v); }
std::string limbs_decimal(int prec, const double* p) {
  return prec == PP_D ? pp::to_decimal_d(p[0])
         : prec == PP_DD ? pp::to_decimal_dd(pp::dd_t{p[0], p[1]})
                         : pp::to_decimal_qd(pp::qd_t{p[0], p[1], p[2], p[3]});
}
// to_double of a level value (xprec.hpp: DD hi + lo; QD ((c3 + c2) + c1) + c0)
double limbs_to_double(int prec, const double* p) {
  return prec == PP_D ? p[0] : prec == PP_DD ? pp::rtod(pp::dd_t{p[0], p[1]}) : pp::rtod(pp::qd_t{p[0], p[1], p[2], p[3]});
}
const char* reason_name(int r) {  // fail_reason_name (tracker.cpp:10-19)
  switch (r) {
    case PP_REASON_NONE: return "converged";
    case PP_REASON_DIVERGED: return "diverged";
    case PP_REASON_STEP_UNDERFLOW: return "step-underflow";
    case PP_REASON_MAX_STEPS: return "max-steps";
    case PP_REASON_SINGULAR: return "singular";
    default: return "no-certificate";
  }
}
}  // namespace

extern "C" {

int pp_solutions_jsonl(const pp_records* rec, int prec, uint32_t dim, const double* gamma, uint64_t seed,
                       const char* command, double wall_ms, uint64_t batches, uint64_t rounds, char* buf,
                       size_t cap, size_t* needed) {
  return guard([&] {
    const int L = limbs_of(prec);
    need(rec != nullptr && L > 0 && gamma != nullptr && needed != nullptr, "pp_solutions_jsonl: bad argument");
    std::string o;
    uint64_t converged = 0, diverged = 0, failed = 0;
    std::vector<double> resid;
    for (uint64_t i = 0; i < rec->count; ++i) {
      const double res = limbs_to_double(prec, rec->residual + i * L);
      const char* cls = rec->status[i] == PP_SUCCESS ? "converged"
                        : rec->reason[i] == PP_REASON_DIVERGED ? "diverged" : "failed";
      if (rec->status[i] == PP_SUCCESS) {
        ++converged;
        resid.push_back(res);
      } else if (rec->reason[i] == PP_REASON_DIVERGED) {
        ++diverged;
      } else {
        ++failed;
      }
      // record_json (polypath_main.cpp:133-150); keys in nlohmann's (sorted) order
      o += "{\"annotation\":\"";
      o += reason_name(rec->reason[i]);
      o += "\",\"newton\":" + std::to_string(rec->newton_iters[i]);
      o += ",\"path\":" + std::to_string(rec->path_id[i]);
      o += ",\"rejections\":" + std::to_string(rec->rejections[i]);
      o += ",\"residual\":";
      put_double(o, res);
      o += ",\"start\":" + std::to_string(rec->path_id[i]);
      o += ",\"status\":\"";
      o += cls;
      o += "\",\"steps\":" + std::to_string(rec->steps[i]);
      o += ",\"type\":\"solution\",\"wall_ms\":";
      put_double(o, wall_ms);
      o += ",\"x\":[";
      for (uint32_t v = 0; v < dim; ++v) {
        const double* z = rec->x + (i * dim + v) * 2 * L;
        o += v ? ",[\"" : "[\"";
        o += limbs_decimal(prec, z);
        o += "\",\"";
        o += limbs_decimal(prec, z + L);
        o += "\"]";
      }
      o += "]}\n";
    }
    // summary (polypath_main.cpp:170-188)
    std::sort(resid.begin(), resid.end());
    o += "{\"batches\":" + std::to_string(batches);
    o += ",\"command\":\"" + std::string(command ? command : "solve") + "\"";
    o += ",\"converged\":" + std::to_string(converged);
    o += ",\"corrector_rounds\":" + std::to_string(rounds);
    o += ",\"diverged\":" + std::to_string(diverged);
    o += ",\"failed\":" + std::to_string(failed);
    o += ",\"gamma\":[";
    put_double(o, limbs_to_double(prec, gamma));
    o += ",";
    put_double(o, limbs_to_double(prec, gamma + L));
    o += "],\"paths\":" + std::to_string(rec->count);
    o += ",\"precision\":\"";
    o += prec == PP_D ? "d" : prec == PP_DD ? "dd" : "qd";
    o += "\"";
    if (!resid.empty()) {
      o += ",\"residual_max\":";
      put_double(o, resid.back());
      o += ",\"residual_median\":";
      put_double(o, resid[resid.size() / 2]);
      o += ",\"residual_min\":";
      put_double(o, resid.front());
    }
    o += ",\"seed\":" + std::to_string(seed);
    o += ",\"type\":\"summary\",\"wall_ms\":";
    put_double(o, wall_ms);
    o += "}\n";
    *needed = o.size() + 1;
    if (buf == nullptr || cap < o.size() + 1) return PP_E_CAPACITY;
    std::memcpy(buf, o.c_str(), o.size() + 1);
    return PP_OK;
  });
}

int pp_bench_eval(const pp_homotopy* h, uint64_t seed, uint32_t batch, uint32_t reps, int device, double* ms,
                  uint64_t* checksum) {
  return guard([&] {
    need(h != nullptr && batch > 0 && ms != nullptr && checksum != nullptr, "pp_bench_eval: bad argument");
    const pp::Plan& plan = h->plan;
    const uint32_t n = plan.dim, np = plan.n_polys, L = plan.L, w = 2 * L;
    // points and t exactly as cmd_bench draws them (polypath_main.cpp:299-319): splitmix64 units
    uint64_t state = seed * 0x9e3779b97f4a7c15ULL + 0x243f6a8885a308d3ULL;
    auto next_unit = [&state]() {
      state += 0x9e3779b97f4a7c15ULL;
      uint64_t z = state;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      z ^= z >> 31;
      return 2.0 * (static_cast<double>(z >> 11) * 0x1p-53) - 1.0;
    };
    std::vector<double> xp(static_cast<size_t>(batch) * n * w, 0.0), tp(static_cast<size_t>(batch) * L, 0.0);
    for (uint32_t j = 0; j < batch; ++j) {
      for (uint32_t v = 0; v < n; ++v) {
        xp[(static_cast<size_t>(v) * w + 0) * batch + j] = next_unit();      // re, limb 0 (R{double})
        xp[(static_cast<size_t>(v) * w + L) * batch + j] = next_unit();      // im, limb 0
      }
      tp[j] = 0.5 * (next_unit() + 1.0);  // R{0.5 * (u + 1)}: limb 0
    }
    std::vector<double> sys(static_cast<size_t>(batch) * np * w), jac(static_cast<size_t>(batch) * np * n * w);
    pp_homotopy* hm = const_cast<pp_homotopy*>(h);
    *ms = pp::device_bench_eval(plan, hm->on(device), batch, xp.data(), tp.data(), reps, sys.data(), jac.data(), device);
    // fnv1a over ws.sys.raw() then ws.jac.raw() (polypath_main.cpp:275-282, 341-342)
    uint64_t hsh = 0xcbf29ce484222325ULL;
    auto fnv = [&hsh](const std::vector<double>& d) {
      const unsigned char* p = reinterpret_cast<const unsigned char*>(d.data());
      for (size_t i = 0; i < d.size() * sizeof(double); ++i) {
        hsh ^= p[i];
        hsh *= 0x100000001b3ULL;
      }
    };
    fnv(sys);
    fnv(jac);
    *checksum = hsh;
    return PP_OK;
  });
}

int pp_to_decimal(int prec, const double* limbs, char* buf, size_t cap) {
  return guard([&] {
    need(limbs_of(prec) > 0 && limbs != nullptr, "pp_to_decimal: bad argument");
    const std::string t = limbs_decimal(prec, limbs);
    if (buf == nullptr || cap < t.size() + 1) return PP_E_CAPACITY;
    std::memcpy(buf, t.c_str(), t.size() + 1);
    return PP_OK;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// testing hooks (include/pp200_testing.h): host-side arithmetic of xprec.cuh, for bitwise
// comparison against the reference build.  Op codes match oracle/ref_harness.cpp ref_arith.
// ---------------------------------------------------------------------------------------------
namespace {
template <class R>
R get_r(const double* p) {
  R v;
  for (int l = 0; l < pp::level<R>::L; ++l) pp::level<R>::set(v, l, p[l]);
  return v;
}
template <class R>
void put_r(const R& v, double* p) {
  for (int l = 0; l < pp::level<R>::L; ++l) p[l] = pp::level<R>::get(v, l);
}
template <class R>
pp::cx<R> get_c(const double* p) {
  return {get_r<R>(p), get_r<R>(p + pp::level<R>::L)};
}
template <class R>
void put_c(const pp::cx<R>& z, double* p) {
  put_r(z.re, p);
  put_r(z.im, p + pp::level<R>::L);
}
template <class R>
int arith(int op, const double* a, const double* b, double* out) {
  using namespace pp;
  const R x = get_r<R>(a), y = get_r<R>(b);
  switch (op) {
    case 0: put_r(radd(x, y), out); break;
    case 1: put_r(rsub(x, y), out); break;
    case 2: put_r(rmul(x, y), out); break;
    case 3: put_r(rmuld(x, b[0]), out); break;
    case 4: put_r(rdiv(x, y), out); break;
    case 5: put_r(rsqrt(x), out); break;
    case 6: out[0] = rcmp(x, y); break;
    case 7: out[0] = rtod(x); break;
    case 8: put_c(cmul(get_c<R>(a), get_c<R>(b)), out); break;
    case 9: put_c(cdiv(get_c<R>(a), get_c<R>(b)), out); break;
    case 10: put_r(cabsr(get_c<R>(a)), out); break;
    default: return PP_E_INVALID;
  }
  return PP_OK;
}
}  // namespace

extern "C" {

int pp_test_arith(int prec, int op, const double* a, const double* b, double* out) {
  switch (prec) {
    case PP_D: return arith<double>(op, a, b, out);
    case PP_DD: return arith<pp::dd_t>(op, a, b, out);
    case PP_QD: return arith<pp::qd_t>(op, a, b, out);
    default: return PP_E_INVALID;
  }
}

int pp_test_parse_decimal(int prec, const char* s, double* out) {
  switch (prec) {
    case PP_D: return pp::parse_decimal_d(s, out[0]) ? PP_OK : PP_E_PARSE;
    case PP_DD: {
      pp::dd_t v;
      if (!pp::parse_decimal_dd(s, v)) return PP_E_PARSE;
      out[0] = v.hi, out[1] = v.lo;
      return PP_OK;
    }
    case PP_QD: {
      pp::qd_t v;
      if (!pp::parse_decimal_qd(s, v)) return PP_E_PARSE;
      out[0] = v.c0, out[1] = v.c1, out[2] = v.c2, out[3] = v.c3;
      return PP_OK;
    }
    default: return PP_E_INVALID;
  }
}

int pp_test_to_decimal(int prec, const double* in, char* buf, size_t cap) {
  std::string s = prec == PP_D ? pp::to_decimal_d(in[0])
                  : prec == PP_DD ? pp::to_decimal_dd(pp::dd_t{in[0], in[1]})
                                  : pp::to_decimal_qd(pp::qd_t{in[0], in[1], in[2], in[3]});
  if (s.size() + 1 > cap) return PP_E_CAPACITY;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return PP_OK;
}

int pp_fp64_peak(int device, double* ops_per_s) {
  return guard([&] {
    need(ops_per_s != nullptr, "pp_fp64_peak: null argument");
    *ops_per_s = pp::device_fp64_peak(device);
    return PP_OK;
  });
}

// plan coefficients (per term: c_start then c_target, 2L each) for cross-checks against the
// reference's build_plan
int pp_test_plan_coeffs(const pp_homotopy* h, double* out, size_t cap) {
  if (h == nullptr || cap < h->plan.coeff.size()) return PP_E_CAPACITY;
  std::copy(h->plan.coeff.begin(), h->plan.coeff.end(), out);
  return PP_OK;
}

int pp_test_plan_tables(const pp_homotopy* h, int which, uint32_t* out, size_t cap, size_t* count) {
  if (h == nullptr || count == nullptr) return PP_E_INVALID;
  const pp::Plan& p = h->plan;
  const std::vector<uint32_t>* v = which == 0 ? &p.term_slot : which == 1 ? &p.acc_off : which == 2 ? &p.acc_idx
                                   : which == 3 ? &p.pos : nullptr;
  std::vector<uint32_t> ti;
  if (which == 4) {
    ti.assign(p.term_info.begin(), p.term_info.end());
    v = &ti;
  }
  if (v == nullptr) return PP_E_INVALID;
  *count = v->size();
  if (out == nullptr || cap < v->size()) return PP_E_CAPACITY;
  std::copy(v->begin(), v->end(), out);
  return PP_OK;
}

// doubles formatted as the JSON records print them (json_number.cpp), newline-separated
int pp_test_json_doubles(const double* v, size_t n, char* buf, size_t cap, size_t* needed) {
  std::string o;
  for (size_t i = 0; i < n; ++i) {
    pp::json_double(o, v[i]);
    o += '\n';
  }
  if (needed) *needed = o.size() + 1;
  if (buf == nullptr || cap < o.size() + 1) return PP_E_CAPACITY;
  std::memcpy(buf, o.c_str(), o.size() + 1);
  return PP_OK;
}

// PathBatch::set_prediction + newton_correct (tracker.hpp:135-136, tracker.cpp:216-274) on the device
int pp_test_newton(const pp_homotopy* h, const pp_track_config* cfg, uint32_t batch, const double* t, double* x,
                   uint32_t* iters, uint8_t* corrected, uint8_t* singular, int device) {
  int rc = pp_track_config_validate(cfg);
  if (rc != PP_OK) return rc;
  return guard([&] {
    need(h != nullptr && (batch == 0 || (t && x && iters && corrected && singular)), "pp_test_newton: null argument");
    pp_homotopy* hm = const_cast<pp_homotopy*>(h);
    pp::device_newton(hm->plan, hm->on(device), *cfg, batch, t, x, iters, corrected, singular, device);
    return PP_OK;
  });
}

}  // extern "C"
