// xprec.cuh -- double, double-double and quad-double real/complex arithmetic for sm_100a and
// for the host, reproducing the reference's operation sequence exactly so that every result is
// bitwise identical to polypath's CPU code (reference: proj/include/polypath/xprec.hpp:18-541,
// proj/include/polypath/complex.hpp:8-107).
//
// Exactness rules.  The reference is compiled with -ffp-contract=off (proj/CMakeLists.txt:14) and
// calls std::fma only in two_prod (xprec.hpp:40) and DD*double (xprec.hpp:233).  On the device every
// binary64 operation below goes through an _rn intrinsic (__dadd_rn, __dmul_rn, __fma_rn,
// __ddiv_rn, __dsqrt_rn), which the compiler never contracts or reassociates; on the host the same
// source is compiled with -ffp-contract=off.  Both round to nearest-even, so both agree with the
// reference bit for bit.  Quad-double addition merges limbs in a data-dependent order
// (xprec.hpp:325-382); here the merge is a sorting network on the limbs' magnitudes that emits the
// same sequence whenever the operands' limbs are ordered (every renormalised value), with the
// step-by-step merge over register queues for any other operand (qdi::add_i).
#pragma once

#include <cmath>
#include <cstdint>

#if defined(__CUDACC__)
#define PP_UNROLL _Pragma("unroll")
#define PP_HD __host__ __device__ __forceinline__
// quad-double operations are 100-250 binary64 instructions each; they are real calls on the
// device so that kernels built from them stay compact (code size, compile time, I-cache)
#define PP_QD_FN static __host__ __device__ __noinline__
// the bodies of the hot quad-double operations, inlined into the complex operations below
#define PP_QD_INL static __host__ __device__ __forceinline__
#else
#define PP_QD_INL inline
#define PP_HD inline
#define PP_QD_FN inline
#define PP_UNROLL
#endif

// host-only operation counter for the work model (scripts/count_ops.cpp defines PP_COUNT_OPS)
#if defined(PP_COUNT_OPS) && !defined(__CUDA_ARCH__)
extern unsigned long long pp_op_count;
#define PP_COUNT() (++pp_op_count)
#else
#define PP_COUNT() ((void)0)
#endif

namespace pp {

// ---------------------------------------------------------------------------------------------
// binary64 primitives
// ---------------------------------------------------------------------------------------------
PP_HD double f_add(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  PP_COUNT(); return a + b;
#endif
}
PP_HD double f_sub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  PP_COUNT(); return a - b;
#endif
}
PP_HD double f_mul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  PP_COUNT(); return a * b;
#endif
}
PP_HD double f_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  PP_COUNT(); return std::fma(a, b, c);
#endif
}
PP_HD double f_div(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __ddiv_rn(a, b);
#else
  PP_COUNT(); return a / b;
#endif
}
PP_HD double f_sqrt(double a) {
#if defined(__CUDA_ARCH__)
  return __dsqrt_rn(a);
#else
  PP_COUNT(); return std::sqrt(a);
#endif
}
PP_HD double f_abs(double a) { return std::fabs(a); }
PP_HD bool f_isinf(double a) {
#if defined(__CUDA_ARCH__)
  return isinf(a);
#else
  return std::isinf(a);
#endif
}
// std::max(a, b) semantics: returns a unless a < b (NaN in b is ignored, NaN in a sticks)
PP_HD double f_max(double a, double b) { return (a < b) ? b : a; }

// ---------------------------------------------------------------------------------------------
// error-free transforms (xprec.hpp:23-42)
// ---------------------------------------------------------------------------------------------
PP_HD double quick_two_sum(double a, double b, double& err) {
  double s = f_add(a, b);
  err = f_sub(b, f_sub(s, a));
  return s;
}
PP_HD double two_sum(double a, double b, double& err) {
  double s = f_add(a, b);
  double bb = f_sub(s, a);
  err = f_add(f_sub(a, f_sub(s, bb)), f_sub(b, bb));
  return s;
}
PP_HD double two_prod(double a, double b, double& err) {
  double p = f_mul(a, b);
  err = f_fma(a, b, -p);
  return p;
}

// ---------------------------------------------------------------------------------------------
// double-double (xprec.hpp:181-291)
// ---------------------------------------------------------------------------------------------
struct dd_t {
  double hi, lo;
};

PP_HD dd_t dd_make(double h) { return dd_t{h, 0.0}; }
PP_HD dd_t dd_norm(double hi, double lo) {
  double e;
  double s = quick_two_sum(hi, lo, e);
  return dd_t{s, e};
}
PP_HD dd_t rneg(dd_t a) { return dd_t{-a.hi, -a.lo}; }
PP_HD dd_t radd(dd_t a, dd_t b) {
  double e1, e2;
  double s = two_sum(a.hi, b.hi, e1);
  double t = two_sum(a.lo, b.lo, e2);
  e1 = f_add(e1, t);
  s = quick_two_sum(s, e1, e1);
  e1 = f_add(e1, e2);
  return dd_norm(s, e1);
}
PP_HD dd_t radd(dd_t a, double b) {
  double e;
  double s = two_sum(a.hi, b, e);
  e = f_add(e, a.lo);
  return dd_norm(s, e);
}
PP_HD dd_t rsub(dd_t a, dd_t b) { return radd(a, rneg(b)); }
PP_HD dd_t rmul(dd_t a, dd_t b) {
  double e;
  double p = two_prod(a.hi, b.hi, e);
  double cross = f_add(f_mul(a.hi, b.lo), f_mul(a.lo, b.hi));
  double low = f_add(e, f_add(cross, f_mul(a.lo, b.lo)));
  return dd_norm(p, low);
}
PP_HD dd_t rmuld(dd_t a, double b) {
  double e;
  double p = two_prod(a.hi, b, e);
  double low = f_fma(a.lo, b, e);
  return dd_norm(p, low);
}
PP_HD dd_t rdiv(dd_t a, dd_t b) {
  // the reference throws std::domain_error on b == 0 (xprec.hpp:240-241); the tracker never
  // divides by an exact zero (rank test, strictly increasing history t), so no check here
  double q1 = f_div(a.hi, b.hi);
  dd_t r = rsub(a, rmuld(b, q1));
  double q2 = f_div(r.hi, b.hi);
  r = rsub(r, rmuld(b, q2));
  double q3 = f_div(r.hi, b.hi);
  double e;
  double s = quick_two_sum(q1, q2, e);
  return radd(dd_t{s, e}, q3);
}
PP_HD int rcmp(dd_t a, dd_t b) {
  if (a.hi < b.hi) return -1;
  if (a.hi > b.hi) return 1;
  if (a.lo < b.lo) return -1;
  if (a.lo > b.lo) return 1;
  return 0;
}
PP_HD dd_t rabs(dd_t a) { return a.hi < 0.0 ? rneg(a) : a; }
PP_HD double rtod(dd_t a) { return f_add(a.hi, a.lo); }
PP_HD dd_t rsqrt(dd_t a) {
  if (a.hi == 0.0 && a.lo == 0.0) return dd_t{0.0, 0.0};
  double x = f_div(1.0, f_sqrt(a.hi));
  double ax = f_mul(a.hi, x);
  dd_t ax2 = rmul(dd_make(ax), dd_make(ax));
  double e;
  double s = two_sum(ax, f_mul(rsub(a, ax2).hi, f_mul(x, 0.5)), e);
  return dd_t{s, e};
}

// ---------------------------------------------------------------------------------------------
// quad-double (xprec.hpp:297-541)
// ---------------------------------------------------------------------------------------------
struct qd_t {
  double c0, c1, c2, c3;
};

PP_HD qd_t qd_make(double x) { return qd_t{x, 0.0, 0.0, 0.0}; }
PP_HD qd_t qd_from_dd(dd_t x) { return qd_t{x.hi, x.lo, 0.0, 0.0}; }

namespace qdi {

PP_HD void three_sum(double& a, double& b, double& c) {
  double t1, t2, t3;
  t1 = two_sum(a, b, t2);
  a = two_sum(c, t1, t3);
  b = two_sum(t2, t3, c);
}
PP_HD void three_sum2(double& a, double& b, double c) {
  double t1, t2, t3;
  t1 = two_sum(a, b, t2);
  a = two_sum(c, t1, t3);
  b = f_add(t2, t3);
}

// 4-limb renormalisation (xprec.hpp:80-105)
PP_HD qd_t renorm(double c0, double c1, double c2, double c3) {
  if (f_isinf(c0)) return qd_t{c0, c1, c2, c3};
  double s0, s1, s2 = 0.0, s3 = 0.0;
  s0 = quick_two_sum(c2, c3, c3);
  s0 = quick_two_sum(c1, s0, c2);
  c0 = quick_two_sum(c0, s0, c1);
  s0 = c0;
  s1 = c1;
  if (s1 != 0.0) {
    s1 = quick_two_sum(s1, c2, s2);
    if (s2 != 0.0)
      s2 = quick_two_sum(s2, c3, s3);
    else
      s1 = quick_two_sum(s1, c3, s2);
  } else {
    s0 = quick_two_sum(s0, c2, s1);
    if (s1 != 0.0)
      s1 = quick_two_sum(s1, c3, s2);
    else
      s0 = quick_two_sum(s0, c3, s1);
  }
  return qd_t{s0, s1, s2, s3};
}

// 5-limb renormalisation (xprec.hpp:107-155)
PP_QD_INL qd_t renorm5_i(double c0, double c1, double c2, double c3, double c4) {
  if (f_isinf(c0)) return qd_t{c0, c1, c2, c3};
  double s0, s1, s2 = 0.0, s3 = 0.0;
  s0 = quick_two_sum(c3, c4, c4);
  s0 = quick_two_sum(c2, s0, c3);
  s0 = quick_two_sum(c1, s0, c2);
  c0 = quick_two_sum(c0, s0, c1);
  s0 = c0;
  s1 = c1;
  if (s1 != 0.0) {
    s1 = quick_two_sum(s1, c2, s2);
    if (s2 != 0.0) {
      s2 = quick_two_sum(s2, c3, s3);
      if (s3 != 0.0)
        s3 = f_add(s3, c4);
      else
        s2 = quick_two_sum(s2, c4, s3);
    } else {
      s1 = quick_two_sum(s1, c3, s2);
      if (s2 != 0.0)
        s2 = quick_two_sum(s2, c4, s3);
      else
        s1 = quick_two_sum(s1, c4, s2);
    }
  } else {
    s0 = quick_two_sum(s0, c2, s1);
    if (s1 != 0.0) {
      s1 = quick_two_sum(s1, c3, s2);
      if (s2 != 0.0)
        s2 = quick_two_sum(s2, c4, s3);
      else
        s1 = quick_two_sum(s1, c4, s2);
    } else {
      s0 = quick_two_sum(s0, c3, s1);
      if (s1 != 0.0)
        s1 = quick_two_sum(s1, c4, s2);
      else
        s0 = quick_two_sum(s0, c4, s1);
    }
  }
  return qd_t{s0, s1, s2, s3};
}
PP_QD_FN qd_t renorm(double c0, double c1, double c2, double c3, double c4) { return renorm5_i(c0, c1, c2, c3, c4); }

// merge step of the accurate addition (xprec.hpp:158-173); returns (emit, s)
PP_HD double three_accum(double& a, double& b, double c) {
  double s;
  s = two_sum(b, c, b);
  s = two_sum(a, s, a);
  bool za = (a != 0.0);
  bool zb = (b != 0.0);
  if (za && zb) return s;
  if (!zb) {
    b = a;
    a = s;
  } else {
    a = s;
  }
  return 0.0;
}

// Register queue over the unconsumed limbs of one operand: head() is the next limb in
// decreasing-magnitude order; pop() shifts.  Replaces the reference's a.limb[i++] indexing.
struct LimbQueue {
  double q0, q1, q2, q3;
  int n;
  PP_HD double pop() {
    double t = q0;
    q0 = q1;
    q1 = q2;
    q2 = q3;
    q3 = 0.0;
    --n;
    return t;
  }
};

// the reference's selection rule: a exhausted -> b; b exhausted -> a; |a_i| > |b_j| -> a; else b
PP_HD double take(LimbQueue& a, LimbQueue& b) {
  bool from_a = (a.n > 0) && (b.n == 0 || f_abs(a.q0) > f_abs(b.q0));
  return from_a ? a.pop() : b.pop();
}

PP_HD void put(double& x0, double& x1, double& x2, double& x3, int k, double s) {
  if (k == 0) x0 = s;
  else if (k == 1) x1 = s;
  else if (k == 2) x2 = s;
  else x3 = s;
}

}  // namespace qdi

PP_HD qd_t rneg(qd_t a) { return qd_t{-a.c0, -a.c1, -a.c2, -a.c3}; }

// accurate merge-based addition (xprec.hpp:325-382)
namespace qdi {
// the accumulation over the merged limbs m0..m7 (the reference's loop after its merge)
PP_HD qd_t accumulate_merged(double m0, double m1, double m2, double m3, double m4, double m5, double m6,
                             double m7) {
  double v0;
  const double u0 = quick_two_sum(m0, m1, v0);
  double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0, x4 = 0.0;
  double u = u0, v = v0;
  int k = 0;
  const double m[6] = {m2, m3, m4, m5, m6, m7};
PP_UNROLL
  for (int step = 0; step < 6; ++step) {
    const double t = m[step];
    if (k < 4) {
      double s = qdi::three_accum(u, v, t);
      if (s != 0.0) {
        qdi::put(x0, x1, x2, x3, k, s);
        ++k;
        if (k == 4) x4 = f_add(u, v);
      }
    } else {
      x4 = f_add(x4, t);
    }
  }
  if (k < 4) {
    qdi::put(x0, x1, x2, x3, k, u);
    if (k < 3)
      qdi::put(x0, x1, x2, x3, k + 1, v);
    else
      x4 = v;
  }
  return qdi::renorm5_i(x0, x1, x2, x3, x4);
}

// The reference's merge, step by step over two limb queues: correct for any limbs (unsorted,
// NaN), but on the GPU every step shifts both queues under predicates.
PP_QD_INL qd_t add_seq_i(qd_t a, qd_t b) {
  qdi::LimbQueue qa{a.c0, a.c1, a.c2, a.c3, 4};
  qdi::LimbQueue qb{b.c0, b.c1, b.c2, b.c3, 4};
  double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0, x4 = 0.0;
  double u = qdi::take(qa, qb);
  double v = qdi::take(qa, qb);
  u = quick_two_sum(u, v, v);
  int k = 0;
  // the six remaining limbs: while fewer than four outputs exist they feed the accumulator,
  // afterwards they fold into the fifth channel (the reference's tail loop, after x4 = u + v)
PP_UNROLL
  for (int step = 0; step < 6; ++step) {
    double t = qdi::take(qa, qb);
    if (k < 4) {
      double s = qdi::three_accum(u, v, t);
      if (s != 0.0) {
        qdi::put(x0, x1, x2, x3, k, s);
        ++k;
        if (k == 4) x4 = f_add(u, v);
      }
    } else {
      x4 = f_add(x4, t);
    }
  }
  if (k < 4) {
    // both operands exhausted with fewer than four outputs
    qdi::put(x0, x1, x2, x3, k, u);
    if (k < 3)
      qdi::put(x0, x1, x2, x3, k + 1, v);
    else
      x4 = v;
  }
  return qdi::renorm5_i(x0, x1, x2, x3, x4);
}
}  // namespace qdi
PP_QD_FN qd_t radd_seq(qd_t a, qd_t b) { return qdi::add_seq_i(a, b); }

namespace qdi {
// compare-exchange of the merge key: x goes first iff |x| > |y|, or |x| == |y| and x's tag is lower
PP_HD void merge_cx(double& x, int& tx, double& y, int& ty) {
  const double ax = f_abs(x), ay = f_abs(y);
  const bool first = (ax > ay) | ((ax == ay) & (tx < ty));
  const double lo = first ? y : x;
  const int tlo = first ? ty : tx;
  x = first ? x : y;
  tx = first ? tx : ty;
  y = lo;
  ty = tlo;
}

// The same addition with the merge done by a network.  When both operands' limbs are ordered by
// non-increasing magnitude (every renormalised value), the reference's merge -- take a_i while
// |a_i| > |b_j|, else b_j -- emits the limbs in the order of the key (|x| descending; among equal
// magnitudes b's limbs before a's, each operand's in index order).  Tagging b_j with j and a_i with
// 4 + i makes that key a total order, so Batcher's odd-even merge of the two sorted runs (9
// compare-exchanges, 3 levels) yields the identical sequence.  Any other operand (unordered limbs,
// NaN) takes the step-by-step merge.  tests/native/qd_add_check.cpp compares the two bit for bit;
// building with -DPP_QD_ADD_NET=0 uses the step-by-step merge everywhere (A/B).
#ifndef PP_QD_ADD_NET
#define PP_QD_ADD_NET 1
#endif
PP_QD_INL qd_t add_i(qd_t a, qd_t b) {
  if (!PP_QD_ADD_NET) return qdi::add_seq_i(a, b);
  const bool sorted = (f_abs(a.c0) >= f_abs(a.c1)) & (f_abs(a.c1) >= f_abs(a.c2)) & (f_abs(a.c2) >= f_abs(a.c3)) &
                      (f_abs(b.c0) >= f_abs(b.c1)) & (f_abs(b.c1) >= f_abs(b.c2)) & (f_abs(b.c2) >= f_abs(b.c3));
  if (!sorted) return radd_seq(a, b);
  double w0 = a.c0, w1 = a.c1, w2 = a.c2, w3 = a.c3, w4 = b.c0, w5 = b.c1, w6 = b.c2, w7 = b.c3;
  int t0 = 4, t1 = 5, t2 = 6, t3 = 7, t4 = 0, t5 = 1, t6 = 2, t7 = 3;
  merge_cx(w0, t0, w4, t4);
  merge_cx(w1, t1, w5, t5);
  merge_cx(w2, t2, w6, t6);
  merge_cx(w3, t3, w7, t7);
  merge_cx(w2, t2, w4, t4);
  merge_cx(w3, t3, w5, t5);
  merge_cx(w1, t1, w2, t2);
  merge_cx(w3, t3, w4, t4);
  merge_cx(w5, t5, w6, t6);
  return accumulate_merged(w0, w1, w2, w3, w4, w5, w6, w7);
}
}  // namespace qdi
PP_QD_FN qd_t radd(qd_t a, qd_t b) { return qdi::add_i(a, b); }

PP_QD_FN qd_t radd(qd_t a, double b) {
  double e;
  double c0 = two_sum(a.c0, b, e);
  double c1 = two_sum(a.c1, e, e);
  double c2 = two_sum(a.c2, e, e);
  double c3 = two_sum(a.c3, e, e);
  return qdi::renorm(c0, c1, c2, c3, e);
}
PP_HD qd_t rsub(qd_t a, qd_t b) { return radd(a, rneg(b)); }

PP_QD_FN qd_t rmuld(qd_t a, double b) {
  double q0, q1, q2;
  double p0 = two_prod(a.c0, b, q0);
  double p1 = two_prod(a.c1, b, q1);
  double p2 = two_prod(a.c2, b, q2);
  double p3 = f_mul(a.c3, b);
  double s0 = p0;
  double s2;
  double s1 = two_sum(q0, p1, s2);
  qdi::three_sum(s2, q1, p2);
  qdi::three_sum2(q1, q2, p3);
  double s3 = q1;
  double s4 = f_add(q2, p2);
  return qdi::renorm(s0, s1, s2, s3, s4);
}

// symmetric accurate product (xprec.hpp:420-480)
namespace qdi {
PP_QD_INL qd_t mul_i(qd_t a, qd_t b) {
  double q0;
  double p0 = two_prod(a.c0, b.c0, q0);

  double xe1, ye1;
  double x1 = two_prod(a.c0, b.c1, xe1);
  double y1 = two_prod(a.c1, b.c0, ye1);
  double cr1e;
  double cr1 = two_sum(x1, y1, cr1e);
  double h1e;
  double h1 = two_sum(cr1, q0, h1e);

  double xe2, ye2;
  double x2 = two_prod(a.c0, b.c2, xe2);
  double y2 = two_prod(a.c2, b.c0, ye2);
  double cr2e;
  double cr2 = two_sum(x2, y2, cr2e);
  double q12e;
  double q12 = two_sum(xe1, ye1, q12e);
  double dge;
  double dg = two_prod(a.c1, b.c1, dge);

  double e1, e2, e3, e4;
  double v1 = two_sum(h1e, cr1e, e1);
  double v2 = two_sum(q12, cr2, e2);
  double v3 = two_sum(v1, v2, e3);
  double s2 = two_sum(v3, dg, e4);

  double xe3, ye3, xe4, ye4;
  double x3 = two_prod(a.c0, b.c3, xe3);
  double y3 = two_prod(a.c3, b.c0, ye3);
  double cr3e;
  double cr3 = two_sum(x3, y3, cr3e);
  double x4 = two_prod(a.c1, b.c2, xe4);
  double y4 = two_prod(a.c2, b.c1, ye4);
  double cr4e;
  double cr4 = two_sum(x4, y4, cr4e);
  double q22e;
  double q22 = two_sum(xe2, ye2, q22e);

  double f1, f2, f3, f4, f5, f6, f7, f8, f9;
  double t1 = two_sum(e1, e2, f1);
  double t2 = two_sum(e3, e4, f2);
  double t3 = two_sum(q12e, cr2e, f3);
  double t4 = two_sum(q22, dge, f4);
  double t5 = two_sum(cr3, cr4, f5);
  double t6 = two_sum(t1, t2, f6);
  double t7 = two_sum(t3, t4, f7);
  double t8 = two_sum(t6, t7, f8);
  double s3 = two_sum(t8, t5, f9);

  // u^4 tail: the reference's left-to-right '+' chain ((((G1 + G2) + f9) + G3) + G4) + G5
  double g12 = f_add(f_add(f_add(f1, f2), f_add(f3, f4)), f_add(f_add(f5, f6), f_add(f7, f8)));
  double acc = f_add(g12, f9);
  acc = f_add(acc, f_add(f_add(q22e, cr3e), cr4e));
  acc = f_add(acc, f_add(f_add(xe3, ye3), f_add(xe4, ye4)));
  acc = f_add(acc, f_add(f_add(f_mul(a.c1, b.c3), f_mul(a.c3, b.c1)), f_mul(a.c2, b.c2)));
  return qdi::renorm5_i(p0, h1, s2, s3, acc);
}
}  // namespace qdi
PP_QD_FN qd_t rmul(qd_t a, qd_t b) { return qdi::mul_i(a, b); }

PP_QD_FN qd_t rdiv(qd_t a, qd_t b) {
  double q0 = f_div(a.c0, b.c0);
  qd_t r = rsub(a, rmuld(b, q0));
  double q1 = f_div(r.c0, b.c0);
  r = rsub(r, rmuld(b, q1));
  double q2 = f_div(r.c0, b.c0);
  r = rsub(r, rmuld(b, q2));
  double q3 = f_div(r.c0, b.c0);
  r = rsub(r, rmuld(b, q3));
  double q4 = f_div(r.c0, b.c0);
  return qdi::renorm(q0, q1, q2, q3, q4);
}

PP_HD int rcmp(qd_t a, qd_t b) {
  if (a.c0 < b.c0) return -1;
  if (a.c0 > b.c0) return 1;
  if (a.c1 < b.c1) return -1;
  if (a.c1 > b.c1) return 1;
  if (a.c2 < b.c2) return -1;
  if (a.c2 > b.c2) return 1;
  if (a.c3 < b.c3) return -1;
  if (a.c3 > b.c3) return 1;
  return 0;
}
PP_HD qd_t rabs(qd_t a) { return a.c0 < 0.0 ? rneg(a) : a; }
PP_HD double rtod(qd_t a) { return f_add(f_add(f_add(a.c3, a.c2), a.c1), a.c0); }
PP_QD_FN qd_t rsqrt(qd_t a) {
  if (a.c0 == 0.0 && a.c1 == 0.0 && a.c2 == 0.0 && a.c3 == 0.0) return qd_make(0.0);
  qd_t r = qd_make(f_div(1.0, f_sqrt(a.c0)));
  qd_t h{f_mul(a.c0, 0.5), f_mul(a.c1, 0.5), f_mul(a.c2, 0.5), f_mul(a.c3, 0.5)};
PP_UNROLL
  for (int it = 0; it < 3; ++it) {
    // r += (0.5 - h*(r*r)) * r, with double - QD == (-QD) + double (xprec.hpp:392)
    qd_t corr = radd(rneg(rmul(h, rmul(r, r))), 0.5);
    r = radd(r, rmul(corr, r));
  }
  return rmul(r, a);
}

// ---------------------------------------------------------------------------------------------
// plain double as a level (precision_traits<double>)
// ---------------------------------------------------------------------------------------------
PP_HD double rneg(double a) { return -a; }
PP_HD double radd(double a, double b) { return f_add(a, b); }
PP_HD double rsub(double a, double b) { return f_sub(a, b); }
PP_HD double rmul(double a, double b) { return f_mul(a, b); }
PP_HD double rmuld(double a, double b) { return f_mul(a, b); }
PP_HD double rdiv(double a, double b) { return f_div(a, b); }
PP_HD int rcmp(double a, double b) { return a < b ? -1 : (a > b ? 1 : 0); }
PP_HD double rabs(double a) { return f_abs(a); }
PP_HD double rtod(double a) { return a; }
PP_HD double rsqrt(double a) { return f_sqrt(a); }

// ---------------------------------------------------------------------------------------------
// level traits: limb count, construction from double, limb access
// ---------------------------------------------------------------------------------------------
template <class R>
struct level;

template <>
struct level<double> {
  static constexpr int L = 1;
  static constexpr int tag = 0;
  PP_HD static double from(double x) { return x; }
  PP_HD static double get(const double& v, int) { return v; }
  PP_HD static void set(double& v, int, double x) { v = x; }
};
template <>
struct level<dd_t> {
  static constexpr int L = 2;
  static constexpr int tag = 1;
  PP_HD static dd_t from(double x) { return dd_t{x, 0.0}; }
  PP_HD static double get(const dd_t& v, int i) { return i == 0 ? v.hi : v.lo; }
  PP_HD static void set(dd_t& v, int i, double x) {
    if (i == 0) v.hi = x;
    else v.lo = x;
  }
};
template <>
struct level<qd_t> {
  static constexpr int L = 4;
  static constexpr int tag = 2;
  PP_HD static qd_t from(double x) { return qd_t{x, 0.0, 0.0, 0.0}; }
  PP_HD static double get(const qd_t& v, int i) {
    return i == 0 ? v.c0 : (i == 1 ? v.c1 : (i == 2 ? v.c2 : v.c3));
  }
  PP_HD static void set(qd_t& v, int i, double x) {
    if (i == 0) v.c0 = x;
    else if (i == 1) v.c1 = x;
    else if (i == 2) v.c2 = x;
    else v.c3 = x;
  }
};

template <class R>
PP_HD R rfrom(double x) {
  return level<R>::from(x);
}

// QD -> level narrowing (xprec.hpp:602-622, convert<To>(QD))
template <class R>
PP_HD R narrow_qd(qd_t x);
template <>
PP_HD double narrow_qd<double>(qd_t x) {
  return rtod(x);
}
template <>
PP_HD dd_t narrow_qd<dd_t>(qd_t x) {
  double lo = f_add(f_add(x.c3, x.c2), x.c1);
  return dd_norm(x.c0, lo);
}
template <>
PP_HD qd_t narrow_qd<qd_t>(qd_t x) {
  return x;
}

// ---------------------------------------------------------------------------------------------
// complex (complex.hpp:8-107)
// ---------------------------------------------------------------------------------------------
template <class R>
struct cx {
  R re, im;
};

template <class R>
PP_HD cx<R> cmake(R re, R im) {
  return cx<R>{re, im};
}
template <class R>
PP_HD cx<R> czero() {
  return cx<R>{rfrom<R>(0.0), rfrom<R>(0.0)};
}
template <class R>
PP_HD cx<R> cone() {
  return cx<R>{rfrom<R>(1.0), rfrom<R>(0.0)};
}
template <class R>
PP_HD cx<R> cneg(cx<R> a) {
  return cx<R>{rneg(a.re), rneg(a.im)};
}
template <class R>
PP_HD cx<R> cadd(cx<R> a, cx<R> b) {
  return cx<R>{radd(a.re, b.re), radd(a.im, b.im)};
}
template <class R>
PP_HD cx<R> csub(cx<R> a, cx<R> b) {
  return cx<R>{rsub(a.re, b.re), rsub(a.im, b.im)};
}
// 4-mul / 2-add product, no fused operations (complex.hpp:37-40)
template <class R>
PP_HD cx<R> cmul(cx<R> a, cx<R> b) {
  return cx<R>{rsub(rmul(a.re, b.re), rmul(a.im, b.im)), radd(rmul(a.re, b.im), rmul(a.im, b.re))};
}
// scaling by a real at the same level (complex.hpp:43-46)
template <class R>
PP_HD cx<R> cmulr(cx<R> a, R s) {
  return cx<R>{rmul(a.re, s), rmul(a.im, s)};
}
// scaling by a double (complex.hpp:53-54; for R = double identical to cmulr)
template <class R>
PP_HD cx<R> cmuld(cx<R> a, double s) {
  return cx<R>{rmuld(a.re, s), rmuld(a.im, s)};
}
template <class R>
PP_HD cx<R> cconj(cx<R> a) {
  return cx<R>{a.re, rneg(a.im)};
}
template <class R>
PP_HD R cabs2(cx<R> a) {
  return radd(rmul(a.re, a.re), rmul(a.im, a.im));
}
template <class R>
PP_HD R cabsr(cx<R> a) {
  return rsqrt(cabs2(a));
}
// to_double(cabs(z)), the tracker's norm primitive (tracker.cpp:250, 262-263)
template <class R>
PP_HD double cabsd(cx<R> a) {
  return rtod(cabsr(a));
}
// PP_QD_CPLX_CALLS=1 builds the complex quad-double operations below as single calls with their
// real operations inlined.  Measured slower on the B200 (katsura-12 qd, 4,096 paths: 21.6 s
// against 20.4 s with one call per real operation; the inlined bodies cost registers and I-cache
// more than the extra scheduling freedom gains), so it is off by default.
#ifndef PP_QD_CPLX_CALLS
#define PP_QD_CPLX_CALLS 0
#endif
#if PP_QD_CPLX_CALLS
// complex quad-double: one call per complex operation, with the real operations inlined inside it,
// so that the independent real products and sums of a complex operation are scheduled together
// (the same operations in the same order as the templates above; exact-match overloads win)
PP_QD_FN cx<qd_t> cmul(cx<qd_t> a, cx<qd_t> b) {
  return cx<qd_t>{qdi::add_i(qdi::mul_i(a.re, b.re), rneg(qdi::mul_i(a.im, b.im))),
                  qdi::add_i(qdi::mul_i(a.re, b.im), qdi::mul_i(a.im, b.re))};
}
PP_QD_FN cx<qd_t> cadd(cx<qd_t> a, cx<qd_t> b) { return cx<qd_t>{qdi::add_i(a.re, b.re), qdi::add_i(a.im, b.im)}; }
PP_QD_FN cx<qd_t> csub(cx<qd_t> a, cx<qd_t> b) {
  return cx<qd_t>{qdi::add_i(a.re, rneg(b.re)), qdi::add_i(a.im, rneg(b.im))};
}
PP_QD_FN cx<qd_t> cmulr(cx<qd_t> a, qd_t s) { return cx<qd_t>{qdi::mul_i(a.re, s), qdi::mul_i(a.im, s)}; }
PP_QD_FN qd_t cabs2(cx<qd_t> a) { return qdi::add_i(qdi::mul_i(a.re, a.re), qdi::mul_i(a.im, a.im)); }
#endif

// Smith division (complex.hpp:92-107); b != 0 is the caller's invariant
template <class R>
PP_HD cx<R> cdiv(cx<R> a, cx<R> b) {
  if (rcmp(rabs(b.re), rabs(b.im)) >= 0) {
    R r = rdiv(b.im, b.re);
    R den = radd(b.re, rmul(b.im, r));
    return cx<R>{rdiv(radd(a.re, rmul(a.im, r)), den), rdiv(rsub(a.im, rmul(a.re, r)), den)};
  }
  R r = rdiv(b.re, b.im);
  R den = radd(b.im, rmul(b.re, r));
  return cx<R>{rdiv(radd(rmul(a.re, r), a.im), den), rdiv(rsub(rmul(a.im, r), a.re), den)};
}

}  // namespace pp
