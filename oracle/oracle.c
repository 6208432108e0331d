/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain-C restatement of the reference
 * tracker, one path at a time.  Every function cites the reference code it restates
 * (paths relative to /root/reference/proj).  Built with -ffp-contract=off like the reference
 * (CMakeLists.txt:14); fma() is called exactly where the reference calls std::fma.
 *
 * Structure deliberately differs from the product: the monomial stage interprets an explicit
 * step list (set_one / copy / mul over value, derivative, acc and aux slots) built exactly as
 * evaldiff.cpp:90-168 builds it, while the CUDA kernels run a fused register schedule; the
 * history is a shifted array as in tracker.cpp:276-291, the product uses a ring buffer.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double v[4]; } real;
typedef struct { real re, im; } cplx;

static int LV = 2; /* limbs of the current level */

/* ---------------- error-free transforms (include/polypath/xprec.hpp:23-42) ---------------- */
static double qsum(double a, double b, double* e) {
  double s = a + b;
  *e = b - (s - a);
  return s;
}
static double tsum(double a, double b, double* e) {
  double s = a + b, bb = s - a;
  *e = (a - (s - bb)) + (b - bb);
  return s;
}
static double tprod(double a, double b, double* e) {
  double p = a * b;
  *e = fma(a, b, -p);
  return p;
}

/* ---------------- double-double (xprec.hpp:181-291) ---------------- */
static real dd(double h, double l) {
  real r = {{h, l, 0, 0}};
  return r;
}
static real dd_norm(double h, double l) {
  double e, s = qsum(h, l, &e);
  return dd(s, e);
}
static real dd_add(real a, real b) {
  double e1, e2, s = tsum(a.v[0], b.v[0], &e1), t = tsum(a.v[1], b.v[1], &e2);
  e1 += t;
  s = qsum(s, e1, &e1);
  e1 += e2;
  return dd_norm(s, e1);
}
static real dd_add_d(real a, double b) {
  double e, s = tsum(a.v[0], b, &e);
  e += a.v[1];
  return dd_norm(s, e);
}
static real dd_mul(real a, real b) {
  double e, p = tprod(a.v[0], b.v[0], &e);
  double cross = a.v[0] * b.v[1] + a.v[1] * b.v[0];
  double low = e + (cross + a.v[1] * b.v[1]);
  return dd_norm(p, low);
}
static real dd_mul_d(real a, double b) {
  double e, p = tprod(a.v[0], b, &e);
  return dd_norm(p, fma(a.v[1], b, e));
}
static real dd_neg(real a) { return dd(-a.v[0], -a.v[1]); }
static real dd_div(real a, real b) {
  double q1 = a.v[0] / b.v[0];
  real r = dd_add(a, dd_neg(dd_mul_d(b, q1)));
  double q2 = r.v[0] / b.v[0];
  r = dd_add(r, dd_neg(dd_mul_d(b, q2)));
  double q3 = r.v[0] / b.v[0], e, s = qsum(q1, q2, &e);
  return dd_add_d(dd(s, e), q3);
}
static real dd_sqrt(real a) {
  if (a.v[0] == 0.0 && a.v[1] == 0.0) return dd(0, 0);
  double x = 1.0 / sqrt(a.v[0]), ax = a.v[0] * x, e;
  real ax2 = dd_mul(dd(ax, 0), dd(ax, 0));
  double s = tsum(ax, dd_add(a, dd_neg(ax2)).v[0] * (x * 0.5), &e);
  return dd(s, e);
}

/* ---------------- quad-double (xprec.hpp:60-541) ---------------- */
static real qd(double a, double b, double c, double d) {
  real r = {{a, b, c, d}};
  return r;
}
static void three_sum(double* a, double* b, double* c) {
  double t1, t2, t3;
  t1 = tsum(*a, *b, &t2);
  *a = tsum(*c, t1, &t3);
  *b = tsum(t2, t3, c);
}
static void three_sum2(double* a, double* b, double c) {
  double t1, t2, t3;
  t1 = tsum(*a, *b, &t2);
  *a = tsum(c, t1, &t3);
  *b = t2 + t3;
}
/* xprec.hpp:107-155 */
static real renorm5(double c0, double c1, double c2, double c3, double c4) {
  double s0, s1, s2 = 0.0, s3 = 0.0;
  if (isinf(c0)) return qd(c0, c1, c2, c3);
  s0 = qsum(c3, c4, &c4);
  s0 = qsum(c2, s0, &c3);
  s0 = qsum(c1, s0, &c2);
  c0 = qsum(c0, s0, &c1);
  s0 = c0;
  s1 = c1;
  if (s1 != 0.0) {
    s1 = qsum(s1, c2, &s2);
    if (s2 != 0.0) {
      s2 = qsum(s2, c3, &s3);
      if (s3 != 0.0) s3 += c4;
      else s2 = qsum(s2, c4, &s3);
    } else {
      s1 = qsum(s1, c3, &s2);
      if (s2 != 0.0) s2 = qsum(s2, c4, &s3);
      else s1 = qsum(s1, c4, &s2);
    }
  } else {
    s0 = qsum(s0, c2, &s1);
    if (s1 != 0.0) {
      s1 = qsum(s1, c3, &s2);
      if (s2 != 0.0) s2 = qsum(s2, c4, &s3);
      else s1 = qsum(s1, c4, &s2);
    } else {
      s0 = qsum(s0, c3, &s1);
      if (s1 != 0.0) s1 = qsum(s1, c4, &s2);
      else s0 = qsum(s0, c4, &s1);
    }
  }
  return qd(s0, s1, s2, s3);
}
/* xprec.hpp:158-173 */
static double three_accum(double* a, double* b, double c) {
  double s = tsum(*b, c, b);
  s = tsum(*a, s, a);
  int za = *a != 0.0, zb = *b != 0.0;
  if (za && zb) return s;
  if (!zb) {
    *b = *a;
    *a = s;
  } else {
    *a = s;
  }
  return 0.0;
}
/* merge order of the accurate addition: the larger head first, b on ties (xprec.hpp:330-375) */
static double pick(const real* a, const real* b, int* i, int* j) {
  if (*i >= 4) return b->v[(*j)++];
  if (*j >= 4) return a->v[(*i)++];
  if (fabs(a->v[*i]) > fabs(b->v[*j])) return a->v[(*i)++];
  return b->v[(*j)++];
}
/* xprec.hpp:325-382 */
static real qd_add(real a, real b) {
  int i = 0, j = 0, k = 0;
  double x[4] = {0, 0, 0, 0}, x4 = 0.0, u, v, s, t;
  u = pick(&a, &b, &i, &j);
  v = pick(&a, &b, &i, &j);
  u = qsum(u, v, &v);
  while (k < 4) {
    if (i >= 4 && j >= 4) {
      x[k] = u;
      if (k < 3) x[++k] = v;
      else x4 = v;
      u = v = 0.0;
      break;
    }
    t = pick(&a, &b, &i, &j);
    s = three_accum(&u, &v, t);
    if (s != 0.0) x[k++] = s;
  }
  if (k >= 4) x4 = u + v;
  while (i < 4 || j < 4) x4 += pick(&a, &b, &i, &j);
  return renorm5(x[0], x[1], x[2], x[3], x4);
}
static real qd_neg(real a) { return qd(-a.v[0], -a.v[1], -a.v[2], -a.v[3]); }
static real qd_add_d(real a, double b) {
  double e, c0 = tsum(a.v[0], b, &e), c1 = tsum(a.v[1], e, &e), c2 = tsum(a.v[2], e, &e), c3 = tsum(a.v[3], e, &e);
  return renorm5(c0, c1, c2, c3, e);
}
static real qd_mul_d(real a, double b) {
  double q0, q1, q2, s2;
  double p0 = tprod(a.v[0], b, &q0), p1 = tprod(a.v[1], b, &q1), p2 = tprod(a.v[2], b, &q2), p3 = a.v[3] * b;
  double s1 = tsum(q0, p1, &s2);
  three_sum(&s2, &q1, &p2);
  three_sum2(&q1, &q2, p3);
  return renorm5(p0, s1, s2, q1, q2 + p2);
}
/* xprec.hpp:420-480 */
static real qd_mul(real a, real b) {
  const double* A = a.v;
  const double* B = b.v;
  double q0, p0 = tprod(A[0], B[0], &q0);
  double xe1, ye1, cr1e, h1e;
  double x1 = tprod(A[0], B[1], &xe1), y1 = tprod(A[1], B[0], &ye1);
  double cr1 = tsum(x1, y1, &cr1e), h1 = tsum(cr1, q0, &h1e);
  double xe2, ye2, cr2e, q12e, dge;
  double x2 = tprod(A[0], B[2], &xe2), y2 = tprod(A[2], B[0], &ye2);
  double cr2 = tsum(x2, y2, &cr2e), q12 = tsum(xe1, ye1, &q12e), dg = tprod(A[1], B[1], &dge);
  double e1, e2, e3, e4;
  double v1 = tsum(h1e, cr1e, &e1), v2 = tsum(q12, cr2, &e2), v3 = tsum(v1, v2, &e3), s2 = tsum(v3, dg, &e4);
  double xe3, ye3, xe4, ye4, cr3e, cr4e, q22e;
  double x3 = tprod(A[0], B[3], &xe3), y3 = tprod(A[3], B[0], &ye3), cr3 = tsum(x3, y3, &cr3e);
  double x4 = tprod(A[1], B[2], &xe4), y4 = tprod(A[2], B[1], &ye4), cr4 = tsum(x4, y4, &cr4e);
  double q22 = tsum(xe2, ye2, &q22e);
  double f1, f2, f3, f4, f5, f6, f7, f8, f9;
  double t1 = tsum(e1, e2, &f1), t2 = tsum(e3, e4, &f2), t3 = tsum(q12e, cr2e, &f3), t4 = tsum(q22, dge, &f4);
  double t5 = tsum(cr3, cr4, &f5), t6 = tsum(t1, t2, &f6), t7 = tsum(t3, t4, &f7), t8 = tsum(t6, t7, &f8);
  double s3 = tsum(t8, t5, &f9);
  double tail = ((f1 + f2) + (f3 + f4)) + ((f5 + f6) + (f7 + f8)) + f9 + ((q22e + cr3e) + cr4e) +
                ((xe3 + ye3) + (xe4 + ye4)) + ((A[1] * B[3] + A[3] * B[1]) + A[2] * B[2]);
  return renorm5(p0, h1, s2, s3, tail);
}
static real qd_div(real a, real b) {
  double q0 = a.v[0] / b.v[0];
  real r = qd_add(a, qd_neg(qd_mul_d(b, q0)));
  double q1 = r.v[0] / b.v[0];
  r = qd_add(r, qd_neg(qd_mul_d(b, q1)));
  double q2 = r.v[0] / b.v[0];
  r = qd_add(r, qd_neg(qd_mul_d(b, q2)));
  double q3 = r.v[0] / b.v[0];
  r = qd_add(r, qd_neg(qd_mul_d(b, q3)));
  return renorm5(q0, q1, q2, q3, r.v[0] / b.v[0]);
}
static real qd_sqrt(real a) {
  if (a.v[0] == 0.0 && a.v[1] == 0.0 && a.v[2] == 0.0 && a.v[3] == 0.0) return qd(0, 0, 0, 0);
  real r = qd(1.0 / sqrt(a.v[0]), 0, 0, 0);
  real h = qd(a.v[0] * 0.5, a.v[1] * 0.5, a.v[2] * 0.5, a.v[3] * 0.5);
  for (int it = 0; it < 3; ++it) r = qd_add(r, qd_mul(qd_add_d(qd_neg(qd_mul(h, qd_mul(r, r))), 0.5), r));
  return qd_mul(r, a);
}

/* ---------------- the current level ---------------- */
static real R(double x) {
  real r = {{x, 0, 0, 0}};
  return r;
}
static real r_add(real a, real b) {
  if (LV == 1) return R(a.v[0] + b.v[0]);
  return LV == 2 ? dd_add(a, b) : qd_add(a, b);
}
static real r_neg(real a) { return qd(-a.v[0], -a.v[1], -a.v[2], -a.v[3]); }
static real r_sub(real a, real b) {
  if (LV == 1) return R(a.v[0] - b.v[0]);
  return r_add(a, r_neg(b));
}
static real r_mul(real a, real b) {
  if (LV == 1) return R(a.v[0] * b.v[0]);
  return LV == 2 ? dd_mul(a, b) : qd_mul(a, b);
}
static real r_mul_d(real a, double b) {
  if (LV == 1) return R(a.v[0] * b);
  return LV == 2 ? dd_mul_d(a, b) : qd_mul_d(a, b);
}
static real r_div(real a, real b) {
  if (LV == 1) return R(a.v[0] / b.v[0]);
  return LV == 2 ? dd_div(a, b) : qd_div(a, b);
}
static real r_sqrt(real a) {
  if (LV == 1) return R(sqrt(a.v[0]));
  return LV == 2 ? dd_sqrt(a) : qd_sqrt(a);
}
static int r_cmp(real a, real b) {
  for (int l = 0; l < LV; ++l) {
    if (a.v[l] < b.v[l]) return -1;
    if (a.v[l] > b.v[l]) return 1;
  }
  return 0;
}
static double r_tod(real a) {
  if (LV == 1) return a.v[0];
  if (LV == 2) return a.v[0] + a.v[1];
  return ((a.v[3] + a.v[2]) + a.v[1]) + a.v[0];
}
static real r_abs(real a) { return a.v[0] < 0.0 ? r_neg(a) : a; }

/* ---------------- complex (include/polypath/complex.hpp) ---------------- */
static cplx C(real re, real im) {
  cplx z = {re, im};
  return z;
}
static cplx c_zero(void) { return C(R(0), R(0)); }
static cplx c_add(cplx a, cplx b) { return C(r_add(a.re, b.re), r_add(a.im, b.im)); }
static cplx c_sub(cplx a, cplx b) { return C(r_sub(a.re, b.re), r_sub(a.im, b.im)); }
static cplx c_neg(cplx a) { return C(r_neg(a.re), r_neg(a.im)); }
static cplx c_mul(cplx a, cplx b) {
  return C(r_sub(r_mul(a.re, b.re), r_mul(a.im, b.im)), r_add(r_mul(a.re, b.im), r_mul(a.im, b.re)));
}
static cplx c_scale(cplx a, real s) { return C(r_mul(a.re, s), r_mul(a.im, s)); }
static cplx c_scale_d(cplx a, double s) { return C(r_mul_d(a.re, s), r_mul_d(a.im, s)); }
static cplx c_conj(cplx a) { return C(a.re, r_neg(a.im)); }
static real c_abs2(cplx a) { return r_add(r_mul(a.re, a.re), r_mul(a.im, a.im)); }
static real c_abs(cplx a) { return r_sqrt(c_abs2(a)); }
static double c_absd(cplx a) { return r_tod(c_abs(a)); }
static cplx c_div(cplx a, cplx b) { /* complex.hpp:92-107 */
  if (r_cmp(r_abs(b.re), r_abs(b.im)) >= 0) {
    real r = r_div(b.im, b.re), den = r_add(b.re, r_mul(b.im, r));
    return C(r_div(r_add(a.re, r_mul(a.im, r)), den), r_div(r_sub(a.im, r_mul(a.re, r)), den));
  }
  real r = r_div(b.re, b.im), den = r_add(b.im, r_mul(b.re, r));
  return C(r_div(r_add(r_mul(a.re, r), a.im), den), r_div(r_sub(r_mul(a.im, r), a.re), den));
}
static double dmax(double a, double b) { return a < b ? b : a; } /* std::max */

static cplx c_load(const double* p) {
  cplx z = c_zero();
  for (int l = 0; l < LV; ++l) {
    z.re.v[l] = p[l];
    z.im.v[l] = p[LV + l];
  }
  return z;
}
static void c_store(double* p, cplx z) {
  for (int l = 0; l < LV; ++l) {
    p[l] = z.re.v[l];
    p[LV + l] = z.im.v[l];
  }
}

/* ---------------- monomial step lists (src/evaldiff.cpp:90-168) ---------------- */
enum { OP_ONE, OP_COPY, OP_MUL };
enum { LOC_NONE, LOC_POINT, LOC_SLOT, LOC_ACC, LOC_AUX };
typedef struct { int op, dst, drow, a, arow, b, brow; } step;

static int emit(step* s, int n, int op, int dst, int drow, int a, int arow, int b, int brow) {
  step t = {op, dst, drow, a, arow, b, brow};
  s[n] = t;
  return n + 1;
}

/* slots: 0 = value, 1 + j = derivative for position j (term-relative) */
static int build_steps(const uint32_t* pos, int k, step* s) {
  int n = 0;
#define VAR(j) ((int)(pos[j] & 0xffffu))
  if (k == 1) {
    n = emit(s, n, OP_COPY, LOC_SLOT, 0, LOC_POINT, VAR(0), LOC_NONE, 0);
    n = emit(s, n, OP_ONE, LOC_SLOT, 1, LOC_NONE, 0, LOC_NONE, 0);
  } else if (k >= 2) {
    n = emit(s, n, OP_COPY, LOC_SLOT, 2, LOC_POINT, VAR(0), LOC_NONE, 0);
    for (int j = 2; j < k; ++j) n = emit(s, n, OP_MUL, LOC_SLOT, 1 + j, LOC_SLOT, j, LOC_POINT, VAR(j - 1));
    n = emit(s, n, OP_MUL, LOC_SLOT, 0, LOC_SLOT, k, LOC_POINT, VAR(k - 1));
    n = emit(s, n, OP_COPY, LOC_ACC, 0, LOC_POINT, VAR(k - 1), LOC_NONE, 0);
    for (int j = k - 2; j >= 1; --j) {
      n = emit(s, n, OP_MUL, LOC_SLOT, 1 + j, LOC_SLOT, 1 + j, LOC_ACC, 0);
      n = emit(s, n, OP_MUL, LOC_ACC, 0, LOC_ACC, 0, LOC_POINT, VAR(j));
    }
    n = emit(s, n, OP_COPY, LOC_SLOT, 1, LOC_ACC, 0, LOC_NONE, 0);
  }
  /* common factor prod x^(e-1), square-and-multiply (evaldiff.cpp:119-161) */
  int init = 0, any = 0;
  for (int j = 0; j < k; ++j) {
    unsigned e = (pos[j] >> 16) - 1u;
    if (e == 0) continue;
    any = 1;
    if (e == 1) {
      n = init ? emit(s, n, OP_MUL, LOC_AUX, 0, LOC_AUX, 0, LOC_POINT, VAR(j))
               : emit(s, n, OP_COPY, LOC_AUX, 0, LOC_POINT, VAR(j), LOC_NONE, 0);
      init = 1;
      continue;
    }
    n = emit(s, n, OP_COPY, LOC_ACC, 0, LOC_POINT, VAR(j), LOC_NONE, 0);
    for (unsigned bits = e; bits != 0;) {
      if (bits & 1u) {
        n = init ? emit(s, n, OP_MUL, LOC_AUX, 0, LOC_AUX, 0, LOC_ACC, 0)
                 : emit(s, n, OP_COPY, LOC_AUX, 0, LOC_ACC, 0, LOC_NONE, 0);
        init = 1;
      }
      bits >>= 1;
      if (bits != 0) n = emit(s, n, OP_MUL, LOC_ACC, 0, LOC_ACC, 0, LOC_ACC, 0);
    }
  }
  if (any)
    for (int q = 0; q <= k; ++q) n = emit(s, n, OP_MUL, LOC_SLOT, q, LOC_SLOT, q, LOC_AUX, 0);
#undef VAR
  return n;
}

/* H and the row-major Jacobian at (x, t) (evaldiff.cpp:259-374 for one column) */
static void eval_point(const oracle_plan* p, const cplx* x, real t, cplx* sys, cplx* jac) {
  const int dim = p->dim;
  real u = r_sub(R(1.0), t); /* evaldiff.hpp:198-201 */
  for (int i = 0; i < p->n_polys; ++i) sys[i] = c_zero();
  for (int i = 0; i < p->n_polys * dim; ++i) jac[i] = c_zero();
  cplx slot[70];
  step steps[1024];
  for (int i = 0; i < p->n_terms; ++i) {
    const int32_t* ti = p->term_info + 4 * i;
    const int poly = ti[0], k = ti[1];
    const uint32_t* pos = p->pos + ti[2];
    cplx cs = c_load(p->coeff + (size_t)i * 4 * LV), ct = c_load(p->coeff + (size_t)i * 4 * LV + 2 * LV);
    cplx c = C(r_add(r_mul(cs.re, u), r_mul(ct.re, t)), r_add(r_mul(cs.im, u), r_mul(ct.im, t)));
    if (k == 0) {
      sys[poly] = c_add(sys[poly], c);
      continue;
    }
    cplx acc = c_zero(), aux = c_zero();
    int ns = build_steps(pos, k, steps);
    for (int q = 0; q < ns; ++q) {
      const step* st = &steps[q];
      cplx a = c_zero(), b = c_zero(), r;
      if (st->a == LOC_POINT) a = x[st->arow];
      else if (st->a == LOC_SLOT) a = slot[st->arow];
      else if (st->a == LOC_ACC) a = acc;
      else if (st->a == LOC_AUX) a = aux;
      if (st->b == LOC_POINT) b = x[st->brow];
      else if (st->b == LOC_SLOT) b = slot[st->brow];
      else if (st->b == LOC_ACC) b = acc;
      else if (st->b == LOC_AUX) b = aux;
      if (st->op == OP_ONE) r = C(R(1.0), R(0.0));
      else if (st->op == OP_COPY) r = a;
      else r = c_mul(a, b);
      if (st->dst == LOC_SLOT) slot[st->drow] = r;
      else if (st->dst == LOC_ACC) acc = r;
      else aux = r;
    }
    sys[poly] = c_add(sys[poly], c_mul(c, slot[0]));
    for (int j = 0; j < k; ++j) {
      unsigned e = pos[j] >> 16;
      cplx w = c_mul(c, slot[1 + j]);
      if (e != 1) w = c_scale_d(w, (double)e);
      int row = poly * dim + (int)(pos[j] & 0xffffu);
      jac[row] = c_add(jac[row], w);
    }
  }
}

/* mgs_qr + least_squares_solve (include/polypath/linalg.hpp:57-125); a column-major, modified */
static int lsq(int n, cplx* a, const cplx* b, cplx* x) {
  cplx* r = calloc((size_t)n * n, sizeof(cplx));
  cplx* y = calloc((size_t)n, sizeof(cplx));
  for (int i = 0; i < n * n; ++i) r[i] = c_zero();
  real max_norm = R(0);
  for (int j = 0; j < n; ++j) {
    real acc = R(0);
    for (int i = 0; i < n; ++i) acc = r_add(acc, c_abs2(a[j * n + i]));
    real nj = r_sqrt(acc);
    if (r_cmp(nj, max_norm) > 0) max_norm = nj;
  }
  const double tol_d = LV == 1 ? 1e-8 : (LV == 2 ? 1e-16 : 1e-32);
  real tol = r_mul(max_norm, R(tol_d));
  int ok = 1;
  for (int k = 0; k < n && ok; ++k) {
    cplx* ck = a + k * n;
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = 0; i < k; ++i) {
        cplx rik = c_zero();
        for (int q = 0; q < n; ++q) rik = c_add(rik, c_mul(c_conj(a[i * n + q]), ck[q]));
        r[k * n + i] = c_add(r[k * n + i], rik); /* r(i,k), column-major */
        for (int q = 0; q < n; ++q) ck[q] = c_sub(ck[q], c_mul(rik, a[i * n + q]));
      }
    }
    real acc = R(0);
    for (int q = 0; q < n; ++q) acc = r_add(acc, c_abs2(ck[q]));
    real rkk = r_sqrt(acc);
    if (r_cmp(rkk, tol) <= 0) {
      ok = 0;
      break;
    }
    r[k * n + k] = C(rkk, R(0));
    real rinv = r_div(R(1.0), rkk);
    for (int q = 0; q < n; ++q) ck[q] = c_scale(ck[q], rinv);
  }
  if (ok) {
    for (int j = 0; j < n; ++j) {
      cplx acc = c_zero();
      for (int q = 0; q < n; ++q) acc = c_add(acc, c_mul(c_conj(a[j * n + q]), b[q]));
      y[j] = acc;
    }
    for (int j = n - 1; j >= 0; --j) {
      cplx acc = y[j];
      for (int i = j + 1; i < n; ++i) acc = c_sub(acc, c_mul(r[i * n + j], x[i]));
      x[j] = c_div(acc, r[j * n + j]);
    }
  }
  free(r);
  free(y);
  return ok;
}

/* ---------------- exported kernels ---------------- */
int oracle_eval(const oracle_plan* p, const double* x, const double* t, double* sys, double* jac) {
  LV = p->L;
  cplx* xs = malloc(sizeof(cplx) * p->dim);
  cplx* s = malloc(sizeof(cplx) * p->n_polys);
  cplx* j = malloc(sizeof(cplx) * (size_t)p->n_polys * p->dim);
  for (int v = 0; v < p->dim; ++v) xs[v] = c_load(x + v * 2 * LV);
  real tt = R(0);
  for (int l = 0; l < LV; ++l) tt.v[l] = t[l];
  eval_point(p, xs, tt, s, j);
  for (int i = 0; i < p->n_polys; ++i) c_store(sys + i * 2 * LV, s[i]);
  if (jac)
    for (int i = 0; i < p->n_polys * p->dim; ++i) c_store(jac + i * 2 * LV, j[i]);
  free(xs);
  free(s);
  free(j);
  return 0;
}

int oracle_lsq(int L, int n, const double* a, const double* b, double* x) {
  LV = L;
  cplx* A = malloc(sizeof(cplx) * n * n);
  cplx* B = malloc(sizeof(cplx) * n);
  cplx* X = malloc(sizeof(cplx) * n);
  for (int i = 0; i < n * n; ++i) A[i] = c_load(a + i * 2 * L);
  for (int i = 0; i < n; ++i) B[i] = c_load(b + i * 2 * L);
  int ok = lsq(n, A, B, X);
  for (int i = 0; i < n; ++i) c_store(x + i * 2 * L, ok ? X[i] : c_zero());
  free(A);
  free(B);
  free(X);
  return ok;
}

/* ---------------- one path (src/tracker.cpp:135-509) ---------------- */
enum { ST_FAILED = -1, ST_ACTIVE = 0, ST_SUCCESS = 1 };
enum { RS_NONE, RS_DIVERGED, RS_UNDERFLOW, RS_MAXSTEPS, RS_SINGULAR, RS_NOCERT };
#define HIST 5

int oracle_track_path(const oracle_plan* p, const oracle_cfg* c, const double* x0, double* x_out,
                      double* resid_out, int32_t* info) {
  LV = p->L;
  const int n = p->dim;
  cplx* x = malloc(sizeof(cplx) * n);        /* working point (ws.points) */
  cplx* xacc = malloc(sizeof(cplx) * n);     /* accepted point */
  cplx* hx = malloc(sizeof(cplx) * HIST * n);
  cplx* sys = malloc(sizeof(cplx) * n);
  cplx* jac = malloc(sizeof(cplx) * n * n);
  cplx* A = malloc(sizeof(cplx) * n * n);
  cplx* rhs = malloc(sizeof(cplx) * n);
  cplx* dx = malloc(sizeof(cplx) * n);
  real ht[HIST];
  int hist_len = 1, consec = 0, status = ST_ACTIVE, reason = RS_NONE, sing = 0, corrected = 0;
  uint32_t steps = 0, newton = 0, rej = 0;
  /* seed (tracker.cpp:135-153) */
  real t = R(0), h = R(c->h_init), tnext = R(0);
  for (int v = 0; v < n; ++v) xacc[v] = hx[v] = c_load(x0 + v * 2 * LV);
  ht[0] = R(0);

  while (status == ST_ACTIVE) {
    /* predict (tracker.cpp:178-214) */
    tnext = r_add(t, h);
    if (r_cmp(tnext, R(1.0)) >= 0) tnext = R(1.0);
    if (hist_len == 1) {
      for (int v = 0; v < n; ++v) x[v] = hx[v];
    } else {
      real w[HIST];
      for (int i = 0; i < hist_len; ++i) {
        w[i] = R(1.0);
        for (int j = 0; j < hist_len; ++j)
          if (j != i) w[i] = r_mul(w[i], r_div(r_sub(tnext, ht[j]), r_sub(ht[i], ht[j])));
      }
      for (int v = 0; v < n; ++v) {
        cplx acc = c_zero();
        for (int i = 0; i < hist_len; ++i) acc = c_add(acc, c_scale(hx[i * n + v], w[i]));
        x[v] = acc;
      }
    }
    /* newton_correct (tracker.cpp:216-274) */
    corrected = 0;
    sing = 0;
    double xn = 0.0;
    for (int it = 0; it < c->max_newton; ++it) {
      eval_point(p, x, tnext, sys, jac);
      ++newton;
      double resid = 0.0;
      for (int i = 0; i < n; ++i) {
        rhs[i] = c_neg(sys[i]);
        resid = dmax(resid, c_absd(sys[i]));
        for (int w = 0; w < n; ++w) A[w * n + i] = jac[i * n + w];
      }
      if (!lsq(n, A, rhs, dx)) {
        sing = 1;
        break;
      }
      double dxn = 0.0;
      xn = 0.0;
      for (int v = 0; v < n; ++v) {
        x[v] = c_add(x[v], dx[v]);
        dxn = dmax(dxn, c_absd(dx[v]));
        xn = dmax(xn, c_absd(x[v]));
      }
      if (resid <= c->residual_tol && dxn <= c->update_tol * dmax(1.0, xn)) {
        corrected = 1;
        break;
      }
    }
    /* step_control (tracker.cpp:276-317) */
    if (corrected) {
      ++steps;
      if (consec < 255) ++consec;
      t = tnext;
      for (int v = 0; v < n; ++v) xacc[v] = x[v];
      if (hist_len == HIST) {
        for (int i = 0; i + 1 < HIST; ++i) {
          ht[i] = ht[i + 1];
          for (int v = 0; v < n; ++v) hx[i * n + v] = hx[(i + 1) * n + v];
        }
        hist_len = HIST - 1;
      }
      ht[hist_len] = tnext;
      for (int v = 0; v < n; ++v) hx[hist_len * n + v] = x[v];
      ++hist_len;
      if (consec >= c->expand_after) {
        real grown = r_mul_d(h, c->expand);
        h = r_cmp(grown, R(c->h_max)) > 0 ? R(c->h_max) : grown;
      }
    } else {
      ++rej;
      consec = 0;
      h = r_mul_d(h, c->contract);
    }
    /* check_status (tracker.cpp:319-338) */
    double an = 0.0;
    for (int v = 0; v < n; ++v) an = dmax(an, c_absd(xacc[v]));
    if (an > c->divergence_bound) {
      status = ST_FAILED;
      reason = RS_DIVERGED;
    } else if (r_cmp(h, R(c->h_min)) < 0) {
      status = ST_FAILED;
      reason = sing ? RS_SINGULAR : RS_UNDERFLOW;
    } else if (steps > c->max_steps) {
      status = ST_FAILED;
      reason = RS_MAXSTEPS;
    } else if (r_cmp(t, R(1.0)) == 0 && corrected) {
      status = ST_SUCCESS;
    }
  }

  /* finalize (tracker.cpp:402-509) */
  if (status == ST_FAILED && reason != RS_DIVERGED && !(1.0 - r_tod(t) >= 0.01) && hist_len >= 3) {
    double first = 0.0, prev = -1.0, last = 0.0;
    int growing = 1;
    for (int i = 0; i < hist_len; ++i) {
      double nrm = 0.0;
      for (int v = 0; v < n; ++v) nrm = dmax(nrm, c_absd(hx[i * n + v]));
      if (nrm <= prev) growing = 0;
      if (i == 0) first = nrm;
      prev = last = nrm;
    }
    double uf = 1.0 - r_tod(ht[0]), ul = 1.0 - r_tod(ht[hist_len - 1]);
    if (growing && first > 0.0 && ul > 0.0 && uf > ul) {
      double m_est = log(last / first) / log(uf / ul);
      if (last >= 10.0 && m_est >= 0.05) reason = RS_DIVERGED;
    }
  }
  if (status == ST_SUCCESS) {
    for (int v = 0; v < n; ++v) x[v] = xacc[v];
    for (int it = 0; it < 3; ++it) {
      eval_point(p, x, R(1.0), sys, jac);
      for (int i = 0; i < n; ++i) {
        rhs[i] = c_neg(sys[i]);
        for (int w = 0; w < n; ++w) A[w * n + i] = jac[i * n + w];
      }
      if (!lsq(n, A, rhs, dx)) break;
      double dxn = 0.0, xn = 0.0;
      for (int v = 0; v < n; ++v) {
        x[v] = c_add(x[v], dx[v]);
        dxn = dmax(dxn, c_absd(dx[v]));
        xn = dmax(xn, c_absd(x[v]));
      }
      if (dxn <= c->update_tol * dmax(1.0, xn)) break;
    }
    for (int v = 0; v < n; ++v) xacc[v] = x[v];
  }
  eval_point(p, xacc, R(1.0), sys, jac);
  real resid = R(0);
  for (int i = 0; i < n; ++i) {
    real m = c_abs(sys[i]);
    if (r_cmp(m, resid) > 0) resid = m;
  }
  if (status == ST_SUCCESS && r_tod(resid) > 10.0 * c->residual_tol) {
    status = ST_FAILED;
    reason = RS_NOCERT;
  }
  for (int v = 0; v < n; ++v) c_store(x_out + v * 2 * LV, xacc[v]);
  for (int l = 0; l < LV; ++l) resid_out[l] = resid.v[l];
  info[0] = status;
  info[1] = reason;
  info[2] = (int32_t)steps;
  info[3] = (int32_t)newton;
  info[4] = (int32_t)rej;
  free(x);
  free(xacc);
  free(hx);
  free(sys);
  free(jac);
  free(A);
  free(rhs);
  free(dx);
  return 0;
}

int oracle_arith(int L, int op, const double* a, const double* b, double* out) {
  LV = L;
  real x = R(0), y = R(0);
  for (int l = 0; l < L; ++l) {
    x.v[l] = a[l];
    y.v[l] = b[l];
  }
  real r = R(0);
  switch (op) {
    case 0: r = r_add(x, y); break;
    case 1: r = r_sub(x, y); break;
    case 2: r = r_mul(x, y); break;
    case 3: r = r_mul_d(x, b[0]); break;
    case 4: r = r_div(x, y); break;
    case 5: r = r_sqrt(x); break;
    case 6: out[0] = r_cmp(x, y); return 0;
    case 7: out[0] = r_tod(x); return 0;
    case 8: c_store(out, c_mul(c_load(a), c_load(b))); return 0;
    case 9: c_store(out, c_div(c_load(a), c_load(b))); return 0;
    case 10: r = c_abs(c_load(a)); break;
    default: return -1;
  }
  for (int l = 0; l < L; ++l) out[l] = r.v[l];
  return 0;
}
