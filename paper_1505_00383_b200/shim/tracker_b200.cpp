// tracker_b200.cpp -- the reference-side drop-in: polypath::track_all<R> with the reference
// signature (proj/include/polypath/tracker.hpp:166-170), implemented on the B200 library through
// its C ABI (include/pp200.h).  A polypath maintainer compiles this file into the polypath build
// (next to, or instead of, the track_all definition in proj/src/tracker.cpp:511-551) and links
// libpp200.so; every caller of track_all -- the CLI (tools/polypath_main.cpp:223-224, 266-267),
// the tests, the acceptance suite -- then runs on the GPU unchanged.
//
// The definitions below are explicit specializations, i.e. strong symbols: linked together with
// an unmodified tracker.o, whose template instantiations are weak, they take precedence
// (oracle/Makefile builds the reference acceptance suite this way).
//
// Semantics kept: TrackConfig::validate first and std::invalid_argument for an empty start set
// (tracker.cpp:514-516); records sorted by path_id (tracker.cpp:537-538); the ProgressSink is
// invoked synchronously on the calling thread with the reference's StepEvents (tracker.cpp:312-315),
// in batches as the device produces them (the events of one path keep their order).
// Differences in bookkeeping fields only: SolutionSet::batches counts device calls (one per GPU
// used) instead of lockstep cohorts, total_rounds counts device trips (one evaluation + solve per
// busy path each) instead of cohort corrector rounds, and PathRecord::wall_ms is the whole call's
// wall time (the reference stores its cohort's).
//
// Environment: POLYPATH_B200_DEVICE (first CUDA device, default 0) and POLYPATH_B200_DEVICES (how
// many devices to use, default 1; with N > 1 the range is split into N block-cyclic shards tracked
// concurrently, one host thread per GPU, and the records merged).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pp200.h"
#include "polypath/tracker.hpp"

namespace polypath {
namespace {

template <class R>
constexpr int pp_tag() {
  return precision_traits<R>::level == Precision::d ? PP_D : precision_traits<R>::level == Precision::dd ? PP_DD : PP_QD;
}

// a complex value as the C ABI's [re limbs, im limbs]
template <class R>
void put(const Cplx<R>& z, double* p) {
  constexpr int L = precision_traits<R>::limbs;
  for (int l = 0; l < L; ++l) {
    p[l] = get_limb(z.re, l);
    p[L + l] = get_limb(z.im, l);
  }
}
template <class R>
Cplx<R> get(const double* p) {
  constexpr int L = precision_traits<R>::limbs;
  Cplx<R> z{};
  for (int l = 0; l < L; ++l) {
    set_limb(z.re, l, p[l]);
    set_limb(z.im, l, p[L + l]);
  }
  return z;
}

void ok(int rc) {
  if (rc == PP_OK) return;
  if (rc == PP_E_INVALID) throw std::invalid_argument(pp_last_error());
  throw std::runtime_error(std::string("B200 tracker: ") + pp_last_error());
}

struct Handles {
  pp_system *f = nullptr, *g = nullptr;
  pp_homotopy* h = nullptr;
  pp_starts* s = nullptr;
  ~Handles() {
    pp_starts_free(s);
    pp_homotopy_free(h);
    pp_system_free(g);
    pp_system_free(f);
  }
};

// the reference's in-memory PolySystem, term by term (exact: QD coefficients cross as limbs)
pp_system* to_pp(const PolySystem& ps) {
  std::vector<uint32_t> counts, nf, fac;
  std::vector<double> co;
  for (const auto& poly : ps.polys) {
    counts.push_back(static_cast<uint32_t>(poly.size()));
    for (const Term& t : poly) {
      double c[8];
      put<QD>(t.coeff, c);
      co.insert(co.end(), c, c + 8);
      nf.push_back(static_cast<uint32_t>(t.mono.factors.size()));
      for (const auto& [v, e] : t.mono.factors) {
        fac.push_back(v);
        fac.push_back(e);
      }
    }
  }
  pp_system* out = nullptr;
  ok(pp_system_from_terms(ps.dim, static_cast<uint32_t>(ps.polys.size()), counts.data(), nf.data(), fac.data(),
                          co.data(), &out));
  return out;
}

unsigned env_u(const char* name, unsigned dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? static_cast<unsigned>(std::strtoul(v, nullptr, 10)) : dflt;
}

// ProgressSink adapter: the C sink receives batches of pp_step_event; the reference sink is called
// once per event, serialised across the per-GPU threads
struct SinkCtx {
  ProgressSink* sink;
  std::mutex mu;
  std::exception_ptr error;
};
void sink_batch(const pp_step_event* ev, uint64_t n, void* user) {
  auto* c = static_cast<SinkCtx*>(user);
  std::lock_guard<std::mutex> lk(c->mu);
  if (c->error) return;
  try {
    for (uint64_t i = 0; i < n; ++i)
      (*c->sink)(StepEvent{ev[i].path_id, ev[i].t, ev[i].h, ev[i].newton_iters, ev[i].status, ev[i].accepted != 0});
  } catch (...) {
    c->error = std::current_exception();
  }
}

template <class R>
SolutionSet<R> track_on_b200(const HomotopyInstance<R>& h, const StartData<R>& starts, const TrackConfig& cfg,
                             ProgressSink* sink, uint64_t lo, uint64_t hi_in) {
  cfg.validate();  // tracker.cpp:514
  if (starts.count == 0) throw std::invalid_argument("track_all: no start solutions");
  const uint64_t hi = std::min<uint64_t>(starts.count, hi_in);
  SolutionSet<R> out;
  if (lo >= hi) return out;
  auto t0 = std::chrono::steady_clock::now();
  constexpr int L = precision_traits<R>::limbs, tag = pp_tag<R>();
  const uint32_t dim = h.target.dim;

  Handles hd;
  hd.f = to_pp(h.target);
  hd.g = to_pp(h.start);
  std::vector<double> gam(2 * L);
  put(h.gamma, gam.data());
  ok(pp_make_homotopy(hd.f, hd.g, tag, gam.data(), &hd.h));
  if (starts.provenance == StartProvenance::total_degree) {  // the reference's own root tables
    std::vector<double> roots;
    for (const auto& tab : starts.roots)
      for (const auto& z : tab) {
        roots.resize(roots.size() + 2 * L);
        put(z, roots.data() + roots.size() - 2 * L);
      }
    ok(pp_starts_roots(tag, dim, starts.degrees.data(), roots.data(), &hd.s));
  } else {
    std::vector<double> x(starts.count * dim * 2 * L);
    for (uint64_t i = 0; i < starts.count; ++i)
      for (uint32_t v = 0; v < dim; ++v) put(starts.explicit_solutions[i][v], &x[(i * dim + v) * 2 * L]);
    ok(pp_starts_explicit(tag, dim, starts.count, x.data(), &hd.s));
  }
  const pp_track_config c{cfg.residual_tol, cfg.update_tol, cfg.max_newton, cfg.expand_after, cfg.h_init,
                          cfg.h_min, cfg.h_max, cfg.expand, cfg.contract, cfg.divergence_bound, cfg.max_steps,
                          cfg.batch, cfg.workers, 0};

  const unsigned first = env_u("POLYPATH_B200_DEVICE", 0);
  const int avail = pp_device_count();
  unsigned ndev = std::max(1u, env_u("POLYPATH_B200_DEVICES", 1));
  if (avail > 0) ndev = std::min<unsigned>(ndev, static_cast<unsigned>(avail) - std::min<unsigned>(first, avail - 1));
  struct Part {
    std::vector<uint64_t> id;
    std::vector<int8_t> st;
    std::vector<uint8_t> rs;
    std::vector<uint32_t> steps, newton, rej;
    std::vector<double> x, res;
    pp_run_stats stats{};
    int rc = PP_OK;
    std::string err;
  };
  std::vector<Part> parts(ndev);
  SinkCtx sctx{sink, {}, nullptr};
  auto run = [&](unsigned r) {
    Part& p = parts[r];
    pp_shard sh{r, ndev, 64};
    const uint64_t n = pp_shard_size(lo, hi, ndev > 1 ? &sh : nullptr);
    p.id.resize(n);
    p.st.resize(n);
    p.rs.resize(n);
    p.steps.resize(n);
    p.newton.resize(n);
    p.rej.resize(n);
    p.x.resize(n * dim * 2 * L);
    p.res.resize(n * L);
    if (n == 0) return;
    pp_records rec{n, 0, p.id.data(), p.st.data(), p.rs.data(), p.steps.data(), p.newton.data(), p.rej.data(),
                   p.x.data(), p.res.data()};
    p.rc = pp_track_all_ex(hd.h, hd.s, &c, lo, hi, ndev > 1 ? &sh : nullptr, sink ? sink_batch : nullptr,
                           sink ? &sctx : nullptr, static_cast<int>(first + r), &rec, &p.stats);
    if (p.rc != PP_OK) p.err = pp_last_error();
  };
  if (ndev == 1) {
    run(0);
  } else {
    std::vector<std::thread> th;
    for (unsigned r = 0; r < ndev; ++r) th.emplace_back(run, r);
    for (auto& t : th) t.join();
  }
  if (sctx.error) std::rethrow_exception(sctx.error);
  for (const Part& p : parts) {
    if (p.rc == PP_E_INVALID) throw std::invalid_argument(p.err);
    if (p.rc != PP_OK) throw std::runtime_error("B200 tracker: " + p.err);
  }
  const double wall =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  for (const Part& p : parts) {
    out.batches += p.id.empty() ? 0 : 1;
    out.total_rounds = std::max<uint64_t>(out.total_rounds, p.stats.total_rounds);
    for (size_t i = 0; i < p.id.size(); ++i) {
      PathRecord<R> r;
      r.path_id = p.id[i];
      r.status = static_cast<PathStatus>(p.st[i]);
      r.reason = static_cast<FailReason>(p.rs[i]);
      r.stats = PathStats{p.steps[i], p.newton[i], p.rej[i]};
      r.x.resize(dim);
      for (uint32_t v = 0; v < dim; ++v) r.x[v] = get<R>(&p.x[(i * dim + v) * 2 * L]);
      for (int l = 0; l < L; ++l) set_limb(r.residual, l, p.res[i * L + l]);
      r.wall_ms = wall;
      out.paths.push_back(std::move(r));
    }
  }
  if (ndev > 1)
    std::sort(out.paths.begin(), out.paths.end(),
              [](const PathRecord<R>& a, const PathRecord<R>& b) { return a.path_id < b.path_id; });
  if (std::getenv("POLYPATH_B200_TRACE"))
    std::fprintf(stderr, "[pp200] track_all<%s>: %zu paths on %u B200 device(s), %.1f ms\n",
                 precision_traits<R>::name, out.paths.size(), ndev, wall);
  return out;
}

// The device is initialised when the program starts (context, per-thread resources, kernel
// modules: about 1.8 s on a fresh process), as a GPU service does at start-up, rather than inside
// whichever track_all call comes first.  POLYPATH_B200_EAGER_INIT=0 defers it to the first call.
// Without a usable device nothing happens here; track_all then fails loudly (no CPU fallback).
struct EagerInit {
  EagerInit() {
    if (env_u("POLYPATH_B200_EAGER_INIT", 1) == 0 || pp_device_count() <= 0) return;
    const unsigned first = env_u("POLYPATH_B200_DEVICE", 0), n = std::max(1u, env_u("POLYPATH_B200_DEVICES", 1));
    for (unsigned d = first; d < first + n && static_cast<int>(d) < pp_device_count(); ++d) pp_device_init(static_cast<int>(d));
  }
};
const EagerInit g_eager_init;

}  // namespace

template <>
SolutionSet<double> track_all<double>(const HomotopyInstance<double>& h, const StartData<double>& s,
                                      const TrackConfig& cfg, ProgressSink* sink, uint64_t lo, uint64_t hi) {
  return track_on_b200<double>(h, s, cfg, sink, lo, hi);
}
template <>
SolutionSet<DD> track_all<DD>(const HomotopyInstance<DD>& h, const StartData<DD>& s, const TrackConfig& cfg,
                              ProgressSink* sink, uint64_t lo, uint64_t hi) {
  return track_on_b200<DD>(h, s, cfg, sink, lo, hi);
}
template <>
SolutionSet<QD> track_all<QD>(const HomotopyInstance<QD>& h, const StartData<QD>& s, const TrackConfig& cfg,
                              ProgressSink* sink, uint64_t lo, uint64_t hi) {
  return track_on_b200<QD>(h, s, cfg, sink, lo, hi);
}

}  // namespace polypath
