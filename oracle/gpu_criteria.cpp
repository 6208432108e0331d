// TEST INFRASTRUCTURE ONLY.  Acceptance criteria 4 (automatic differentiation) and 6 (least
// squares) of the reference suite (proj/tests/acceptance.cpp:167-256, 354-414) re-run with the
// DEVICE doing the work: every evaluation goes through pp_eval_batch (the CUDA evaluation kernel)
// and every factorisation / solve through pp_lsq_batch_mn (the CUDA Gram-Schmidt solver).  The
// systems, points and matrices come from the reference's own generators with the suite's seeds
// (tests/support/oracles.hpp, conditioned.hpp), and the bounds are the suite's.  In addition the
// device results are compared bit for bit with the reference library's (eval_system_batch,
// mgs_qr / least_squares_solve) on the same inputs.
//
// Built by oracle/Makefile as _ref/gpu_criteria (reference objects + libpp200.so).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "pp200.h"
#include "polypath/evaldiff.hpp"
#include "polypath/homotopy.hpp"
#include "polypath/linalg.hpp"
#include "support/conditioned.hpp"
#include "support/oracles.hpp"

using namespace polypath;
using namespace polypath::testing;

namespace {

int g_fail = 0;

void check(int rc, const char* what) {
  if (rc != PP_OK) {
    std::fprintf(stderr, "%s failed: %s\n", what, pp_last_error());
    std::exit(2);
  }
}

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
  check(pp_system_from_terms(ps.dim, static_cast<uint32_t>(ps.polys.size()), counts.data(), nf.data(), fac.data(),
                             co.data(), &out),
        "pp_system_from_terms");
  return out;
}

// H(x, 1) = f(x) on the device: the homotopy of f with itself, gamma = 1, evaluated at t = 1
// (the coefficients at t = 1 are c_target bitwise, evaldiff.hpp:198-201)
template <class R>
void device_eval_f(const PolySystem& s, const std::vector<std::vector<Cplx<R>>>& pts, std::vector<Cplx<R>>& vals,
                   std::vector<Cplx<R>>& jac) {
  constexpr int L = precision_traits<R>::limbs;
  constexpr int tag = L == 1 ? PP_D : (L == 2 ? PP_DD : PP_QD);
  const uint32_t dim = s.dim, B = static_cast<uint32_t>(pts.size());
  pp_system* f = to_pp(s);
  pp_homotopy* h = nullptr;
  std::vector<double> gam(2 * L, 0.0);
  gam[0] = 1.0;
  check(pp_make_homotopy(f, f, tag, gam.data(), &h), "pp_make_homotopy");
  std::vector<double> x(static_cast<size_t>(B) * dim * 2 * L), t(static_cast<size_t>(B) * L, 0.0);
  for (uint32_t b = 0; b < B; ++b) {
    t[static_cast<size_t>(b) * L] = 1.0;
    for (uint32_t v = 0; v < dim; ++v) put(pts[b][v], &x[(static_cast<size_t>(b) * dim + v) * 2 * L]);
  }
  std::vector<double> sys(static_cast<size_t>(B) * dim * 2 * L), jj(static_cast<size_t>(B) * dim * dim * 2 * L);
  check(pp_eval_batch(h, B, x.data(), t.data(), sys.data(), jj.data(), 0), "pp_eval_batch");
  vals.resize(static_cast<size_t>(B) * dim);
  jac.resize(static_cast<size_t>(B) * dim * dim);
  for (size_t i = 0; i < vals.size(); ++i) vals[i] = get<R>(&sys[i * 2 * L]);
  for (size_t i = 0; i < jac.size(); ++i) jac[i] = get<R>(&jj[i * 2 * L]);
  pp_homotopy_free(h);
  pp_system_free(f);
}

bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

void criterion_4_ad_gpu() {
  auto t0 = std::chrono::steady_clock::now();
  std::mt19937_64 rng(20240831);  // acceptance.cpp:169
  bool ok = true, bitwise = true;
  std::string detail;
  double worst_fd = 0.0, worst_sym = 0.0;
  for (int sys_i = 0; sys_i < 100 && ok; ++sys_i) {
    uint32_t dim = 2 + static_cast<uint32_t>(rng() % 5);
    PolySystem s = random_poly_system(rng, dim, 4, 20 / dim + 2);
    auto x = random_point<double>(rng, dim);

    // all double evaluations of this system in one device batch: x, then x +- h e_v (re, im)
    const double hstep = 6e-6;
    std::vector<std::vector<Cplx<double>>> pts{x};
    for (uint32_t v = 0; v < dim; ++v) {
      auto xp = x, xm = x;
      xp[v].re += hstep;
      xm[v].re -= hstep;
      pts.push_back(xp);
      pts.push_back(xm);
      xp = x;
      xm = x;
      xp[v].im += hstep;
      xm[v].im -= hstep;
      pts.push_back(xp);
      pts.push_back(xm);
    }
    std::vector<Cplx<double>> vals, jacs;
    device_eval_f<double>(s, pts, vals, jacs);
    auto val = [&](size_t b, uint32_t p) { return vals[b * dim + p]; };
    std::vector<Cplx<double>> jac(jacs.begin(), jacs.begin() + dim * dim);  // row p*dim + v

    // the reference's eval_system_batch on the same point: bit for bit
    auto pland = build_plan<double>(s);
    BatchWorkspace<double> wsd(pland, 1);
    wsd.set_point(0, x);
    wsd.set_t(0, 1.0);
    eval_system_batch(pland, wsd, 1);
    for (uint32_t i = 0; i < dim * dim; ++i) {
      Cplx<double> r = wsd.jac.load(i, 0);
      bitwise = bitwise && same_bits(r.re, jac[i].re) && same_bits(r.im, jac[i].im);
    }
    for (uint32_t i = 0; i < dim; ++i) {
      Cplx<double> r = wsd.sys.load(i, 0);
      bitwise = bitwise && same_bits(r.re, val(0, i).re) && same_bits(r.im, val(0, i).im);
    }

    double scale = 1.0;
    for (auto& z : jac) scale = std::max(scale, std::abs(z.re) + std::abs(z.im));
    for (uint32_t v = 0; v < dim && ok; ++v) {
      const size_t bp = 1 + 4 * v, bm = bp + 1, bip = bp + 2, bim = bp + 3;
      for (uint32_t p = 0; p < dim; ++p) {
        double fre = (val(bp, p).re - val(bm, p).re) / (2 * hstep);
        double fim = (val(bp, p).im - val(bm, p).im) / (2 * hstep);
        double err = std::max(std::abs(fre - jac[p * dim + v].re), std::abs(fim - jac[p * dim + v].im)) / scale;
        worst_fd = std::max(worst_fd, err);
        if (err >= 1e-6) ok = false, detail = "finite-difference mismatch";
        fre = (val(bip, p).re - val(bim, p).re) / (2 * hstep);
        fim = (val(bip, p).im - val(bim, p).im) / (2 * hstep);
        Cplx<double> expect{-jac[p * dim + v].im, jac[p * dim + v].re};
        err = std::max(std::abs(fre - expect.re), std::abs(fim - expect.im)) / scale;
        worst_fd = std::max(worst_fd, err);
        if (err >= 1e-6) ok = false, detail = "finite-difference mismatch (imaginary)";
      }
    }
    // dd on the device against the symbolic oracle
    std::vector<Cplx<DD>> xdd(dim);
    for (uint32_t i = 0; i < dim; ++i) xdd[i] = convert_cplx<DD>(x[i]);
    std::vector<Cplx<DD>> valsdd, jacdd;
    device_eval_f<DD>(s, {xdd}, valsdd, jacdd);
    auto jref = jacobian_symbolic<DD>(s, std::span<const Cplx<DD>>(xdd));
    for (size_t i = 0; i < jacdd.size(); ++i) {
      double err = to_double(cabs(jacdd[i] - jref[i])) / scale;
      worst_sym = std::max(worst_sym, err);
      if (err >= 1e-13) ok = false, detail = "symbolic mismatch at dd";
    }
  }
  if (!bitwise) ok = false, detail = "device evaluation differs from the reference's eval_system_batch";
  double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (!ok) ++g_fail;
  std::printf("[%s] gpu criterion  4: AD correctness on the device (%.3f s)  -- worst fd %.2e, worst dd-symbolic %.2e, "
              "double evaluations bitwise equal to the reference: %s%s%s\n",
              ok ? "PASS" : "FAIL", sec, worst_fd, worst_sym, bitwise ? "yes" : "NO", detail.empty() ? "" : "; ",
              detail.c_str());
}

void criterion_6_least_squares_gpu() {
  auto t0 = std::chrono::steady_clock::now();
  std::mt19937_64 rng(86420);  // acceptance.cpp:356
  std::uniform_real_distribution<double> d(-1.0, 1.0);
  bool ok = true, bitwise = true;
  std::string detail;
  double worst_orth = 0.0, worst_ls = 0.0;
  for (int it = 0; it < 100 && ok; ++it) {
    double cond = std::pow(10.0, 6.0 * (static_cast<double>(rng() % 1000) / 1000.0));
    uint32_t n = 3 + static_cast<uint32_t>(rng() % 4);
    uint32_t m = n + static_cast<uint32_t>(rng() % 3);
    auto a = conditioned_matrix<double>(rng, m, n, cond);
    std::vector<Cplx<double>> xtrue(n), b(m);
    for (uint32_t j = 0; j < n; ++j) xtrue[j] = {d(rng), d(rng)};
    for (uint32_t i = 0; i < m; ++i) {
      Cplx<double> acc{};
      for (uint32_t j = 0; j < n; ++j) acc += a.at(i, j) * xtrue[j];
      b[i] = acc;
    }
    // the device: Q, R and the solution in one call
    std::vector<double> ha(static_cast<size_t>(m) * n * 2), hb(m * 2), hx(n * 2), hq(ha.size()),
        hr(static_cast<size_t>(n) * (n + 1));
    for (uint32_t j = 0; j < n; ++j)
      for (uint32_t i = 0; i < m; ++i) put(a.at(i, j), &ha[(static_cast<size_t>(j) * m + i) * 2]);
    for (uint32_t i = 0; i < m; ++i) put(b[i], &hb[i * 2]);
    uint8_t okd = 0;
    check(pp_lsq_batch_mn(PP_D, m, n, 1, ha.data(), hb.data(), hx.data(), &okd, hq.data(), hr.data(), 0),
          "pp_lsq_batch_mn");
    if (!okd) {
      ok = false;
      detail = "unexpected rank failure";
      break;
    }
    auto q = [&](uint32_t r, uint32_t c) { return get<double>(&hq[(static_cast<size_t>(c) * m + r) * 2]); };
    double worst = 0.0;
    for (uint32_t i = 0; i < n; ++i)
      for (uint32_t j = 0; j < n; ++j) {
        Cplx<double> dot{};
        for (uint32_t r = 0; r < m; ++r) dot += conj(q(r, i)) * q(r, j);
        if (i == j) dot.re -= 1.0;
        worst = std::max(worst, std::max(std::abs(dot.re), std::abs(dot.im)));
      }
    worst_orth = std::max(worst_orth, worst / (n * 0x1p-53));
    if (worst >= 50.0 * n * 0x1p-53) ok = false, detail = "orthogonality bound violated";
    // the reference's factorisation and solve on the same input: bit for bit
    QRFactors<double> qr;
    std::vector<Cplx<double>> xr(n);
    if (!mgs_qr(a, qr) || !least_squares_solve<double>(a, b, xr)) bitwise = false;
    for (uint32_t c = 0; c < n && bitwise; ++c) {
      for (uint32_t r = 0; r < m; ++r)
        bitwise = bitwise && same_bits(qr.q.at(r, c).re, q(r, c).re) && same_bits(qr.q.at(r, c).im, q(r, c).im);
      for (uint32_t r = 0; r <= c; ++r) {
        Cplx<double> rd = get<double>(&hr[(r + static_cast<size_t>(c) * (c + 1) / 2) * 2]);
        bitwise = bitwise && same_bits(qr.r.at(r, c).re, rd.re) && same_bits(qr.r.at(r, c).im, rd.im);
      }
      Cplx<double> xd = get<double>(&hx[c * 2]);
      bitwise = bitwise && same_bits(xr[c].re, xd.re) && same_bits(xr[c].im, xd.im);
    }
    auto xref = normal_equations_qd(a, b);
    double err = 0.0, scale = 0.0;
    for (uint32_t j = 0; j < n; ++j) {
      err = std::max(err, to_double(cabs(convert_cplx<QD>(get<double>(&hx[j * 2])) - xref[j])));
      scale = std::max(scale, to_double(cabs(xref[j])));
    }
    worst_ls = std::max(worst_ls, err / scale);
    if (err / scale >= 1e-10) ok = false, detail = "LS error above 1e-10";
  }
  if (!bitwise) ok = false, detail = "device factors differ from the reference's mgs_qr / least_squares_solve";
  double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (!ok) ++g_fail;
  std::printf("[%s] gpu criterion  6: least squares on the device (%.3f s)  -- worst orth %.1f n*u, worst LS rel %.2e, "
              "Q, R and x bitwise equal to the reference: %s%s%s\n",
              ok ? "PASS" : "FAIL", sec, worst_orth, worst_ls, bitwise ? "yes" : "NO", detail.empty() ? "" : "; ",
              detail.c_str());
}

}  // namespace

int main() {
  criterion_4_ad_gpu();
  criterion_6_least_squares_gpu();
  if (g_fail) {
    std::printf("%d gpu criterion(s) FAILED\n", g_fail);
    return 1;
  }
  std::printf("all gpu criteria passed\n");
  return 0;
}
