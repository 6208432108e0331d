// track_impl.cuh -- sm_100a kernels of the many-path tracker.
//
// Design: one CUDA thread owns one path slot.  A slot runs the reference's
// per-path state machine -- predict, up to max_newton corrector iterations, step control,
// status, finalize -- and refills itself from a global atomic start counter when its path ends,
// so paths that finish or diverge release their thread immediately (the reference's compaction,
// tracker.cpp:340-387, without a host round trip).  Every trip performs exactly one "heavy"
// operation per slot -- an evaluation of H and dH/dx at the slot's point followed (in corrector /
// refinement modes) by a least-squares solve -- so all lanes of a warp execute the expensive code
// together even though each lane is at a different place on a different path; only the cheap
// bookkeeping diverges.  A trip is two kernels (ctrl_eval_trip, lsq_trip); when few paths
// remain, tail mode gives each path a whole warp (step_trip, eval_coop, lsq_coop).
//
// Per-path results are bitwise identical to the reference CPU tracker: every floating-point
// operation is the reference's (xprec.cuh), executed in the reference's order per path, and the
// reference's per-path results do not depend on batching (test_tracker.cpp:383-432).
//
// Memory: the working point x is in shared memory and the open Jacobian row in tensor memory
// (or shared memory), both indexed by the instruction tables; the Gram-Schmidt column being
// orthogonalised is in shared memory; slot state, history and the accepted point are global,
// slot-minor planar (element e, limb-plane p, slot s at ((e*P)+p)*S+s: a warp's 32 slots touch
// 32 consecutive doubles, the paper's transposed layout, Table 5/7); the solver's
// working arrays (Jacobian / Q, R, b, Q^H b) are slot-tiled (Tiled<R>).  The Speelpenning prefix
// stack is a dynamically indexed local array (KMAX).
#pragma once

#include <cuda_runtime.h>

#include "kernels.hpp"
#include "xprec.cuh"

// register budgets of the trip kernels (minimum resident 128-thread blocks per SM)
#ifndef PP_LSQ_MINB
#define PP_LSQ_MINB 3
#endif
#ifndef PP_EVAL_MINB
#define PP_EVAL_MINB 1
#endif

namespace pp {
namespace dev {

enum : int { M_IDLE = 0, M_NEWTON = 1, M_REFINE = 2, M_FINAL = 3, M_DONE = 4 };
enum : int { ST_FAILED = -1, ST_ACTIVE = 0, ST_SUCCESS = 1 };
enum : int { RS_NONE = 0, RS_DIVERGED = 1, RS_UNDERFLOW = 2, RS_MAXSTEPS = 3, RS_SINGULAR = 4, RS_NOCERT = 5 };
constexpr int kHist = kHistDepth;

// ---------------------------------------------------------------------------------------------
// planar accessors
// ---------------------------------------------------------------------------------------------
template <class R>
struct Planar {
  static constexpr int L = level<R>::L;
  double* base;
  size_t S;  // stride between planes (slots, or blockDim for shared memory)

  // Offsets are formed in 32 bits (one IMAD per element instead of 64-bit multiplies per plane);
  // device_track checks that every planar array holds fewer than 2^32 doubles.
  __device__ __forceinline__ const double* at(uint32_t first_plane, size_t s) const {
    return base + (first_plane * static_cast<uint32_t>(S) + static_cast<uint32_t>(s));
  }
  __device__ __forceinline__ const double& ld_addr(int e, size_t s) const { return *at(static_cast<uint32_t>(e) * 2 * L, s); }
  __device__ __forceinline__ uint32_t plane_stride() const { return static_cast<uint32_t>(S); }
  __device__ __forceinline__ cx<R> ld(int e, size_t s) const {
    cx<R> z;
    const uint32_t S32 = static_cast<uint32_t>(S);
    const double* p = at(static_cast<uint32_t>(e) * 2 * L, s);
#pragma unroll
    for (int l = 0; l < L; ++l) {
      level<R>::set(z.re, l, p[l * S32]);
      level<R>::set(z.im, l, p[(L + l) * S32]);
    }
    return z;
  }
  __device__ __forceinline__ void st(int e, size_t s, const cx<R>& z) const {
    const uint32_t S32 = static_cast<uint32_t>(S);
    double* p = const_cast<double*>(at(static_cast<uint32_t>(e) * 2 * L, s));
#pragma unroll
    for (int l = 0; l < L; ++l) {
      p[l * S32] = level<R>::get(z.re, l);
      p[(L + l) * S32] = level<R>::get(z.im, l);
    }
  }
  // real-valued elements (L planes each)
  __device__ __forceinline__ R ldr(int e, size_t s) const {
    R v;
    const uint32_t S32 = static_cast<uint32_t>(S);
    const double* p = at(static_cast<uint32_t>(e) * L, s);
#pragma unroll
    for (int l = 0; l < L; ++l) level<R>::set(v, l, p[l * S32]);
    return v;
  }
  __device__ __forceinline__ void str(int e, size_t s, const R& v) const {
    const uint32_t S32 = static_cast<uint32_t>(S);
    double* p = const_cast<double*>(at(static_cast<uint32_t>(e) * L, s));
#pragma unroll
    for (int l = 0; l < L; ++l) p[l * S32] = level<R>::get(v, l);
  }
};

// Slot-tiled layout of the solver's working arrays (Jacobian / Q, R, right-hand side, Q^H b): the
// slots are grouped in tiles of 32 (one warp), and a tile's array is contiguous, element-major,
// plane by plane: element e, plane p of slot s at ((s/32)*E*P + e*P + p)*32 + s%32 for an array
// of E complex elements (P = 2L planes).  A warp access is one 256-byte line as in the planar
// layout, but the element's planes are adjacent lines and all strides are compile-time
// multiples of 256 bytes (DRAM row locality, little address arithmetic).
template <class R>
struct Tiled {
  static constexpr int L = level<R>::L;
  double* base;
  uint32_t E;  // complex elements per slot

  __device__ __forceinline__ double* at(int e, size_t s) const {
    const uint32_t tile = static_cast<uint32_t>(s) >> 5, lane = static_cast<uint32_t>(s) & 31u;
    return base + ((tile * E + static_cast<uint32_t>(e)) * (2 * L)) * 32u + lane;
  }
  __device__ __forceinline__ const double& ld_addr(int e, size_t s) const { return *at(e, s); }
  __device__ __forceinline__ uint32_t plane_stride() const { return 32u; }
  __device__ __forceinline__ cx<R> ld(int e, size_t s) const {
    cx<R> z;
    const double* p = at(e, s);
#pragma unroll
    for (int l = 0; l < L; ++l) {
      level<R>::set(z.re, l, p[l * 32]);
      level<R>::set(z.im, l, p[(L + l) * 32]);
    }
    return z;
  }
  __device__ __forceinline__ void st(int e, size_t s, const cx<R>& z) const {
    double* p = at(e, s);
#pragma unroll
    for (int l = 0; l < L; ++l) {
      p[l * 32] = level<R>::get(z.re, l);
      p[(L + l) * 32] = level<R>::get(z.im, l);
    }
  }
  // the same with an L2 cache policy (createpolicy: evict_last keeps the line, evict_first lets it go)
  __device__ __forceinline__ cx<R> ldp(int e, size_t s, uint64_t pol) const {
    cx<R> z;
    const double* p = at(e, s);
#pragma unroll
    for (int l = 0; l < L; ++l) {
      double a, b;
      asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(a) : "l"(p + l * 32), "l"(pol));
      asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(b) : "l"(p + (L + l) * 32), "l"(pol));
      level<R>::set(z.re, l, a);
      level<R>::set(z.im, l, b);
    }
    return z;
  }
  __device__ __forceinline__ void stp(int e, size_t s, const cx<R>& z, uint64_t pol) const {
    double* p = at(e, s);
#pragma unroll
    for (int l = 0; l < L; ++l) {
      asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p + l * 32), "d"(level<R>::get(z.re, l)), "l"(pol)
                   : "memory");
      asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p + (L + l) * 32), "d"(level<R>::get(z.im, l)),
                   "l"(pol)
                   : "memory");
    }
  }
};

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// load of a plan-table entry: through the read-only path from global memory, or (kSm) a plain
// load from the copy the kernel staged in shared memory
template <bool kSm, class T>
__device__ __forceinline__ T tld(const T* p) {
  if constexpr (kSm) {
    return *p;
  } else {
    return __ldg(p);
  }
}

// uniform (warp-broadcast) load of a complex table entry stored as 2L consecutive doubles
template <class R, bool kSm = false>
__device__ __forceinline__ cx<R> ld_table(const double* p) {
  constexpr int L = level<R>::L;
  cx<R> z;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    level<R>::set(z.re, l, tld<kSm>(p + l));
    level<R>::set(z.im, l, tld<kSm>(p + L + l));
  }
  return z;
}

template <class R>
__device__ __forceinline__ void st_flat(double* p, const cx<R>& z) {
  constexpr int L = level<R>::L;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    p[l] = level<R>::get(z.re, l);
    p[L + l] = level<R>::get(z.im, l);
  }
}

template <class R>
__device__ __forceinline__ cx<R> ld_flat(const double* p) {
  constexpr int L = level<R>::L;
  cx<R> z;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    level<R>::set(z.re, l, __ldg(p + l));
    level<R>::set(z.im, l, __ldg(p + L + l));
  }
  return z;
}

// One term of the plan at the point X (this thread's column xs): the coefficient, monomial and
// sum-stage products of evaldiff.cpp:259-374 for term i.  sys_add(v) receives the term's
// contribution to H_poly (c, or c * value), jac_add(j, var, w) the contribution of its j-th
// variable to dH_poly/dx_var, in the reference's order; jac_pre(var) is called before w is
// computed.  The Speelpenning prefix stack is a
// dynamically indexed array (local memory, L1-resident), so the code stays compact for any KMAX.
template <class R, int KMAX, bool kSm = false, class SysF, class JacF, class PreF>
__device__ __forceinline__ void eval_term(const PlanArgs& pa, int i, const Planar<R>& X, size_t xs, const R& t,
                                          const R& u, int& poly_out, SysF&& sys_add, JacF&& jac_add,
                                          PreF&& jac_pre) {
  constexpr int L = level<R>::L;
  const int4 ti = tld<kSm>(reinterpret_cast<const int4*>(pa.term_info) + i);
  const int k = ti.y, po = ti.z, nb = ti.w & 0xff, bo = ti.w >> 8;
  poly_out = ti.x;

  // coefficient stage: c = c_start*(1-t) + c_target*t (evaldiff.cpp:259-274)
  const double* cp = pa.coeff + static_cast<size_t>(i) * 4 * L;
  const cx<R> cs = ld_table<R, kSm>(cp), ct = ld_table<R, kSm>(cp + 2 * L);
  const cx<R> c{radd(rmul(cs.re, u), rmul(ct.re, t)), radd(rmul(cs.im, u), rmul(ct.im, t))};

  if (k == 0) {  // constants skip the monomial stage (evaldiff.cpp:345-352)
    sys_add(c);
    return;
  }

  // common factor prod x^(e-1) by square-and-multiply (evaldiff.cpp:119-161)
  cx<R> aux = czero<R>();
  if (nb > 0) {
    bool init = false;
    for (int b = 0; b < nb; ++b) {
      const uint32_t be = tld<kSm>(pa.base + bo + b);
      const cx<R> xv = X.ld(static_cast<int>(be & 0xffffu), xs);
      const uint32_t e = be >> 16;
      if (e == 1) {
        aux = init ? cmul(aux, xv) : xv;
        init = true;
        continue;
      }
      cx<R> sq = xv;
      for (uint32_t bits = e; bits != 0;) {
        if (bits & 1u) {
          aux = init ? cmul(aux, sq) : sq;
          init = true;
        }
        bits >>= 1;
        if (bits != 0) sq = cmul(sq, sq);
      }
    }
  }

  const uint32_t* pv = pa.pos + po;
  // derivative contribution w = c*d (scaled by the exponent when e != 1) of variable j
  auto contribute = [&](int j, cx<R> d) {
    const uint32_t pe = tld<kSm>(pv + j);
    jac_pre(static_cast<int>(pe & 0xffffu));  // lets the accumulator fetch its old value early
    if (nb > 0) d = cmul(d, aux);
    cx<R> w = cmul(c, d);
    const uint32_t e = pe >> 16;
    if (e != 1) w = cmuld(w, static_cast<double>(e));
    jac_add(j, static_cast<int>(pe & 0xffffu), w);
  };

  if (k == 1) {
    cx<R> val = X.ld(static_cast<int>(tld<kSm>(pv) & 0xffffu), xs);
    if (nb > 0) val = cmul(val, aux);
    sys_add(cmul(c, val));
    contribute(0, cone<R>());
    return;
  }

  // Speelpenning products (evaldiff.cpp:90-115): prefix P_j = x_p0 ... x_p(j-1) for j < k,
  // value = P_(k-1) x_p(k-1), d_j = P_j * S_(j+1) with the running suffix S.
  cx<R> P[KMAX > 1 ? KMAX : 2];
  cx<R> run = X.ld(static_cast<int>(tld<kSm>(pv) & 0xffffu), xs);
  P[1] = run;
  for (int j = 2; j < k; ++j) {
    run = cmul(run, X.ld(static_cast<int>(tld<kSm>(pv + j - 1) & 0xffffu), xs));
    P[j] = run;
  }
  const cx<R> xlast = X.ld(static_cast<int>(tld<kSm>(pv + k - 1) & 0xffffu), xs);
  cx<R> val = cmul(run, xlast);
  if (nb > 0) val = cmul(val, aux);
  sys_add(cmul(c, val));
  contribute(k - 1, run);  // d_(k-1) = P_(k-1)
  cx<R> acc = xlast;
  for (int j = k - 2; j >= 1; --j) {
    const cx<R> d = cmul(P[j], acc);
    acc = cmul(acc, X.ld(static_cast<int>(tld<kSm>(pv + j) & 0xffffu), xs));
    contribute(j, d);
  }
  contribute(0, acc);  // d_0 = S_1
}

// Open Jacobian row accessors for eval_hj: a shared-memory column of this thread, or this
// thread's lane of tensor memory (TMEM).  The TMEM variant frees the shared memory of the open row
// (half of the evaluation's) so more warps fit on an SM; its tcgen05.ld/st are warp-collective,
// which holds because every lane of a warp walks the same plan (the variable index is uniform).
template <class R>
struct SmemRow {
  Planar<R> P;
  size_t ls;
  __device__ __forceinline__ cx<R> ld(int v) const { return P.ld(v, ls); }
  __device__ __forceinline__ void st(int v, const cx<R>& z) const { P.st(v, ls, z); }
  struct Pending {};
  __device__ __forceinline__ void issue(int, Pending&) const {}
  __device__ __forceinline__ void finish_add(int v, Pending&, const cx<R>& w) const { st(v, cadd(ld(v), w)); }
  __device__ __forceinline__ void drain() const {}
};

template <int W>
struct TmemIO;
template <>
struct TmemIO<4> {
  static __device__ __forceinline__ void ld(uint32_t a, uint32_t* r) {
    asm volatile("{\n tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n tcgen05.wait::ld.sync.aligned;\n}"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a) : "memory");
  }
  static __device__ __forceinline__ void st(uint32_t a, const uint32_t* r) {
    asm volatile("{\n tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n tcgen05.wait::st.sync.aligned;\n}"
                 :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
  }
};
template <>
struct TmemIO<8> {
  static __device__ __forceinline__ void ld(uint32_t a, uint32_t* r) {
    asm volatile("{\n tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 " tcgen05.wait::ld.sync.aligned;\n}"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(a) : "memory");
  }
  static __device__ __forceinline__ void st(uint32_t a, const uint32_t* r) {
    asm volatile("{\n tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
                 " tcgen05.wait::st.sync.aligned;\n}"
                 :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
  }
};
template <>
struct TmemIO<16> {
  static __device__ __forceinline__ void ld(uint32_t a, uint32_t* r) {
    TmemIO<8>::ld(a, r);
    TmemIO<8>::ld(a + 8, r + 8);
  }
  static __device__ __forceinline__ void st(uint32_t a, const uint32_t* r) {
    TmemIO<8>::st(a, r);
    TmemIO<8>::st(a + 8, r + 8);
  }
};

// asynchronous forms: the load's registers become valid at tmem_wait_ld (which takes them as
// operands, so the compiler cannot use them earlier); stores complete at tmem_wait_st
template <int W>
__device__ __forceinline__ void tmem_ld_issue(uint32_t a, uint32_t (&r)[W]) {
  if constexpr (W == 4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a) : "memory");
  } else {
#pragma unroll
    for (int q = 0; q < W / 8; ++q)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[8 * q]), "=r"(r[8 * q + 1]), "=r"(r[8 * q + 2]), "=r"(r[8 * q + 3]), "=r"(r[8 * q + 4]),
                     "=r"(r[8 * q + 5]), "=r"(r[8 * q + 6]), "=r"(r[8 * q + 7])
                   : "r"(a + 8 * q) : "memory");
  }
}
template <int W>
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&r)[W]) {
  if constexpr (W == 4) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3])::"memory");
  } else {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7])::"memory");
#pragma unroll
    for (int q = 1; q < W / 8; ++q)
      asm volatile(""
                   : "+r"(r[8 * q]), "+r"(r[8 * q + 1]), "+r"(r[8 * q + 2]), "+r"(r[8 * q + 3]), "+r"(r[8 * q + 4]),
                     "+r"(r[8 * q + 5]), "+r"(r[8 * q + 6]), "+r"(r[8 * q + 7])::"memory");
  }
}
template <int W>
__device__ __forceinline__ void tmem_st_issue(uint32_t a, const uint32_t (&r)[W]) {
  if constexpr (W == 4) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]),
                 "r"(r[3])
                 : "memory");
  } else {
#pragma unroll
    for (int q = 0; q < W / 8; ++q)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a + 8 * q),
                   "r"(r[8 * q]), "r"(r[8 * q + 1]), "r"(r[8 * q + 2]), "r"(r[8 * q + 3]), "r"(r[8 * q + 4]),
                   "r"(r[8 * q + 5]), "r"(r[8 * q + 6]), "r"(r[8 * q + 7])
                   : "memory");
  }
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <class R>
struct TmemRow {
  static constexpr int L = level<R>::L, W = 4 * level<R>::L;  // 32-bit columns per complex value
  uint32_t base;  // this warp's lane quarter and first column
  __device__ __forceinline__ cx<R> ld(int v) const {
    uint32_t r[W];
    __syncwarp();
    tmem_wait_st();  // an earlier asynchronous store (finish_add) may still be in flight
    TmemIO<W>::ld(base + static_cast<uint32_t>(v) * W, r);
    cx<R> z;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      level<R>::set(z.re, l, __hiloint2double(static_cast<int>(r[2 * l + 1]), static_cast<int>(r[2 * l])));
      level<R>::set(z.im, l, __hiloint2double(static_cast<int>(r[2 * (L + l) + 1]), static_cast<int>(r[2 * (L + l)])));
    }
    return z;
  }
  __device__ __forceinline__ void st(int v, const cx<R>& z) const {
    uint32_t r[W];
    pack(z, r);
    __syncwarp();
    TmemIO<W>::st(base + static_cast<uint32_t>(v) * W, r);
  }
  static __device__ __forceinline__ void pack(const cx<R>& z, uint32_t (&r)[W]) {
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const double a = level<R>::get(z.re, l), b = level<R>::get(z.im, l);
      r[2 * l] = static_cast<uint32_t>(__double2loint(a));
      r[2 * l + 1] = static_cast<uint32_t>(__double2hiint(a));
      r[2 * (L + l)] = static_cast<uint32_t>(__double2loint(b));
      r[2 * (L + l) + 1] = static_cast<uint32_t>(__double2hiint(b));
    }
  }
  static __device__ __forceinline__ cx<R> unpack(const uint32_t (&r)[W]) {
    cx<R> z;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      level<R>::set(z.re, l, __hiloint2double(static_cast<int>(r[2 * l + 1]), static_cast<int>(r[2 * l])));
      level<R>::set(z.im, l, __hiloint2double(static_cast<int>(r[2 * (L + l) + 1]), static_cast<int>(r[2 * (L + l)])));
    }
    return z;
  }
  // read-modify-write of one entry with the load issued early: issue() before the contribution
  // is computed, finish_add() after; the store completes at the next issue() (or drain())
  struct Pending {
    uint32_t r[W];
  };
  __device__ __forceinline__ void issue(int v, Pending& p) const {
    __syncwarp();
    tmem_wait_st();
    tmem_ld_issue<W>(base + static_cast<uint32_t>(v) * W, p.r);
  }
  __device__ __forceinline__ void finish_add(int v, Pending& p, const cx<R>& w) const {
    __syncwarp();
    tmem_wait_ld<W>(p.r);
    uint32_t r[W];
    pack(cadd(unpack(p.r), w), r);
    tmem_st_issue<W>(base + static_cast<uint32_t>(v) * W, r);
  }
  __device__ __forceinline__ void drain() const {
    __syncwarp();
    tmem_wait_st();
  }
};

// Thread-per-path evaluation.  X: the point (shared memory, this thread's column); JR: open
// Jacobian row accumulator (shared); outputs: B[p] = -H_p (the least-squares right-hand side,
// tracker.cpp:249), J[v*n_polys + p]; resid_d = max_p to_double(|H_p|) (tracker.cpp:247-251),
// resid_r = max_p |H_p| at level R (tracker.cpp:488-494).  The coefficient, monomial and sum
// stages of the reference are fused per term; because the plan is polynomial-major
// (evaldiff.cpp:200-236), only one row of H/J is open at a time.
template <class R, int KMAX, bool kSm = false, class GA, class ROW>
__device__ void eval_hj(const PlanArgs& pa, const Planar<R>& X, const ROW& JR, size_t ls,
                        const R& t, const GA& B, const GA& J, size_t gs,
                        double& resid_d, R& resid_r) {
  const int n = pa.n, np = pa.n_polys;
  const cx<R> zero = czero<R>();
  const R u = rsub(rfrom<R>(1.0), t);  // ws.set_t: 1 - t at level R (evaldiff.hpp:198-201)

  for (int v = 0; v < n; ++v) JR.st(v, zero);
  cx<R> sacc = zero;
  resid_d = 0.0;
  resid_r = rfrom<R>(0.0);
  int cur = 0;

  auto flush = [&](int p) {
    B.st(p, gs, cneg(sacc));
    R m = cabsr(sacc);
    resid_d = f_max(resid_d, rtod(m));
    if (rcmp(m, resid_r) > 0) resid_r = m;
    for (int v = 0; v < n; ++v) {
      J.st(v * np + p, gs, JR.ld(v));
      JR.st(v, zero);
    }
    sacc = zero;
  };

  for (int i = 0; i < pa.n_terms; ++i) {
    // terms are polynomial-major: close the rows of the polynomials before this term's
    const int poly = tld<kSm>(pa.term_info + 4 * i);
    while (cur < poly) flush(cur++);
    int p_unused;
    typename ROW::Pending pend;
    eval_term<R, KMAX, kSm>(
        pa, i, X, ls, t, u, p_unused, [&](const cx<R>& v) { sacc = cadd(sacc, v); },
        [&](int, int var, const cx<R>& w) { JR.finish_add(var, pend, w); }, [&](int var) { JR.issue(var, pend); });
  }
  while (cur < np) flush(cur++);
  JR.drain();
}

// ---------------------------------------------------------------------------------------------
// least squares, shared-memory column variant (the one the tracker runs)
// ---------------------------------------------------------------------------------------------
// Same operation sequence as lsq_solve (linalg.hpp:79-125), but the column being
// orthogonalised lives in shared memory (C, this thread's column cs), so every row loop is a
// short rolled loop: the solve needs few registers (high occupancy) and its code stays resident
// in the instruction cache.  While column q_i is being applied, the next column to be read is
// prefetched into L1.  On success dx is left in C (elements 0..n-1).
#ifndef PP_LSQ_UNROLL
#define PP_LSQ_UNROLL 2
#endif
#ifndef PP_LSQ_UNROLL_D
#define PP_LSQ_UNROLL_D 4
#endif
// complex double: cheap arithmetic per row, so more rows (loads) in flight per iteration
template <class R>
struct RowsUnroll {
  static constexpr int value = level<R>::L == 1 ? PP_LSQ_UNROLL_D : PP_LSQ_UNROLL;
};
#define PP_UNROLL_ROWS _Pragma("unroll (RowsUnroll<R>::value)")

// PP_LSQ_PREFETCH: 0 none, 1 into L1, 2 into L2 (the next column to be read)
#ifndef PP_LSQ_PREFETCH
#define PP_LSQ_PREFETCH 0
#endif

// PP_SLOT_TILED: the solver's working arrays (J/Q, R, b, Q^H b) in the slot-tiled layout
#ifndef PP_SLOT_TILED
#define PP_SLOT_TILED 1
#endif
#if PP_SLOT_TILED
#define PP_WORK(ptr, E) Tiled<R>{(ptr), static_cast<uint32_t>(E)}
#else
#define PP_WORK(ptr, E) Planar<R>{(ptr), a.S}
#endif

__device__ __forceinline__ void prefetch_line(const double* p) {
#if PP_LSQ_PREFETCH == 1
  asm volatile("prefetch.L1 [%0];" ::"l"(p));
#elif PP_LSQ_PREFETCH == 2
  asm volatile("prefetch.L2 [%0];" ::"l"(p));
#else
  (void)p;
#endif
}

template <class R, class GA>
__device__ __forceinline__ void prefetch_column(const GA& Q, int col, int n, size_t s) {
#if PP_LSQ_PREFETCH
  constexpr int L = level<R>::L;
  for (int e = 0; e < n; ++e) {
    const double* p = &Q.ld_addr(col * n + e, s);
#pragma unroll
    for (int q = 0; q < 2 * L; ++q) prefetch_line(p + q * Q.plane_stride());
  }
#else
  (void)Q, (void)col, (void)n, (void)s;
#endif
}

// Where the axpy of a projection re-reads q_i: from the solver array itself (NoQCache; L1 / L2 /
// HBM), or from a copy the dot product left in the thread's tensor-memory lane (TmemQCache), so
// that q_i streams from global memory once per projection instead of twice.
struct NoQCache {
  template <class R>
  __device__ __forceinline__ void put(int, const cx<R>&) const {}
  __device__ __forceinline__ void commit() const {}
  template <class R, class GA>
  __device__ __forceinline__ cx<R> get(int, const GA& Q, int e, size_t s) const {
    return Q.ld(e, s);
  }
};

template <class R>
struct TmemQCache {
  static constexpr int W = 4 * level<R>::L;  // 32-bit columns per complex value
  uint32_t base;                             // this warp's lane quarter, first column
  __device__ __forceinline__ void put(int r, const cx<R>& q) const {
    uint32_t v[W];
    TmemRow<R>::pack(q, v);
    __syncwarp();
    tmem_st_issue<W>(base + static_cast<uint32_t>(r) * W, v);
  }
  __device__ __forceinline__ void commit() const {
    __syncwarp();
    tmem_wait_st();
  }
  template <class RR, class GA>
  __device__ __forceinline__ cx<R> get(int r, const GA&, int, size_t) const {
    uint32_t v[W];
    __syncwarp();
    TmemIO<W>::ld(base + static_cast<uint32_t>(r) * W, v);
    return TmemRow<R>::unpack(v);
  }
};

// kFuse: each projection's axpy runs in the same row loop as the next projection's dot product
// (row r of the column is updated, then multiplied into the next sum), so the independent axpy
// rows fill the latency of the sequential sum.  Every operation and every sum order is the
// reference's: the dot product of projection j+1 reads each row after projection j's axpy has
// updated it, exactly as the two separate loops do.
// kHint (slot-tiled Q, fused path): the first half of the columns -- read most often, q_i by all
// later columns in both passes -- are loaded and stored with an L2 evict_last policy, the rest
// with evict_first, so that the most reused columns of all slots stay in L2
template <class R, class GA, class CA, bool kUniform, class QC = NoQCache, bool kFuse = false, bool kHint = false>
__device__ bool lsq_solve_c(int n, int m, double rank_tol, const GA& Q, const GA& Rm, const GA& B, const GA& Y,
                            size_t s, const CA& C, const QC& qc = QC{}) {
  [[maybe_unused]] uint64_t pol_keep = 0, pol_drop = 0;
  if constexpr (kHint) {
    pol_keep = l2_policy_evict_last();
    pol_drop = l2_policy_evict_first();
  }
  const int keep_cols = (n + 1) / 2;
  auto qld = [&](int col, int row) -> cx<R> {
    if constexpr (kHint) {
      return Q.ldp(col * m + row, s, col < keep_cols ? pol_keep : pol_drop);
    } else {
      return Q.ld(col * m + row, s);
    }
  };
  auto qst = [&](int col, int row, const cx<R>& z) {
    if constexpr (kHint) {
      Q.stp(col * m + row, s, z, col < keep_cols ? pol_keep : pol_drop);
    } else {
      Q.st(col * m + row, s, z);
    }
  };
  // m x n (m >= n rows; the tracker's systems are square, m == n): Q column-major, element col*m + row
  const cx<R> zero = czero<R>();
  R max_norm = rfrom<R>(0.0);
  for (int j = 0; j < n; ++j) {
    R acc = rfrom<R>(0.0);
PP_UNROLL_ROWS
    for (int r = 0; r < m; ++r) acc = radd(acc, cabs2(Q.ld(j * m + r, s)));
    const R nj = rsqrt(acc);
    if (rcmp(nj, max_norm) > 0) max_norm = nj;
  }
  const R tol = rmul(max_norm, rfrom<R>(rank_tol));

  // kUniform (warp-collective column storage): a rank-deficient lane does not leave early; it
  // finishes the solve on its own scratch with the result discarded, so the warp stays converged
  bool ok = true;
  for (int k = 0; k < n; ++k) {
PP_UNROLL_ROWS
    for (int r = 0; r < m; ++r) C.st(r, qld(k, r));
    const int rk = k * (k + 1) / 2;
    if (kFuse && k > 0) {
      // the 2k projections of column k in order: pass 0 on q_0 .. q_(k-1), then pass 1
      cx<R> rik = zero;
PP_UNROLL_ROWS
      for (int r = 0; r < m; ++r) {
        const cx<R> q = qld(0, r);  // q_0
        qc.put(r, q);
        rik = cadd(rik, cmul(cconj(q), C.ld(r)));
      }
      for (int j = 0; j < 2 * k; ++j) {
        const int pass = j >= k ? 1 : 0, i = j - pass * k;
        const cx<R> prev = pass == 0 ? zero : Rm.ld(i + rk, s);
        Rm.st(i + rk, s, cadd(prev, rik));
        qc.commit();
        if (j + 1 < 2 * k) {
          const int in = (j + 1) % k;  // the next projection's column
          cx<R> rnext = zero;
PP_UNROLL_ROWS
          for (int r = 0; r < m; ++r) {
            const cx<R> qi = qc.template get<R>(r, Q, i * m + r, s);
            const cx<R> c = csub(C.ld(r), cmul(rik, qi));  // axpy of projection j
            const cx<R> qn = qld(in, r);
            qc.put(r, qn);
            C.st(r, c);
            rnext = cadd(rnext, cmul(cconj(qn), c));  // dot product of projection j + 1
          }
          rik = rnext;
        } else {
PP_UNROLL_ROWS
          for (int r = 0; r < m; ++r) C.st(r, csub(C.ld(r), cmul(rik, qc.template get<R>(r, Q, i * m + r, s))));
        }
      }
    }
    for (int pass = 0; pass < 2 && !kFuse; ++pass) {
      for (int i = 0; i < k; ++i) {
        // next column read: q_(i+1), else q_0 of the second pass, else the next column
        const int nxt = i + 1 < k ? i + 1 : (pass == 0 ? 0 : k + 1);
        if (nxt < n) prefetch_column<R>(Q, nxt, m, s);
        cx<R> rik = zero;
PP_UNROLL_ROWS
        for (int r = 0; r < m; ++r) {
          const cx<R> q = Q.ld(i * m + r, s);
          qc.put(r, q);
          rik = cadd(rik, cmul(cconj(q), C.ld(r)));
        }
        const cx<R> prev = pass == 0 ? zero : Rm.ld(i + rk, s);
        Rm.st(i + rk, s, cadd(prev, rik));
        qc.commit();
PP_UNROLL_ROWS
        for (int r = 0; r < m; ++r) C.st(r, csub(C.ld(r), cmul(rik, qc.template get<R>(r, Q, i * m + r, s))));
      }
    }
    R acc = rfrom<R>(0.0);
PP_UNROLL_ROWS
    for (int r = 0; r < m; ++r) acc = radd(acc, cabs2(C.ld(r)));
    const R rkk = rsqrt(acc);
    if (rcmp(rkk, tol) <= 0) {
      if (!kUniform) return false;
      ok = false;
    }
    Rm.st(k + rk, s, cx<R>{rkk, rfrom<R>(0.0)});
    const R rinv = rdiv(rfrom<R>(1.0), rkk);
    cx<R> y = zero;
PP_UNROLL_ROWS
    for (int r = 0; r < m; ++r) {
      const cx<R> q = cmulr(C.ld(r), rinv);
      qst(k, r, q);
      y = cadd(y, cmul(cconj(q), B.ld(r, s)));  // y_k = <q_k, b> (linalg.hpp:117)
    }
    Y.st(k, s, y);
  }
  // back substitution R x = y (linalg.hpp:118-122); x_j overwrites C_j
  for (int j = n - 1; j >= 0; --j) {
    cx<R> acc = Y.ld(j, s);
    for (int i = j + 1; i < n; ++i) acc = csub(acc, cmul(Rm.ld(j + i * (i + 1) / 2, s), C.ld(i)));
    C.st(j, cdiv(acc, Rm.ld(j + j * (j + 1) / 2, s)));
  }
  return ok;
}

// ---------------------------------------------------------------------------------------------
// slot state (global, SoA): integer fields, path index, level-R scalars, double scalars
// ---------------------------------------------------------------------------------------------
enum : int {
  F_MODE = 0, F_IT, F_RIT, F_LEN, F_HEAD, F_CONSEC, F_CORR, F_SING, F_STATUS, F_REASON,
  F_STEPS, F_NEWTON, F_REJ, F_OK, F_COUNT
};
enum : int { R_T = 0, R_H, R_TNEXT, R_RESID, R_COUNT };     // level-R scalars (planar real)
enum : int { D_RESID = 0, D_DXN, D_XN, D_COUNT };          // double scalars
static_assert(F_COUNT == kIntFields && R_COUNT == kRealFields && D_COUNT == kDblFields, "state layout");

struct SlotInts {
  int32_t* base;
  size_t S;
  __device__ __forceinline__ int32_t& operator()(int f, size_t s) const { return base[f * S + s]; }
};


// ---------------------------------------------------------------------------------------------
// trip kernel 2 (thread per path): least-squares Newton update for corrector / refinement slots
// ---------------------------------------------------------------------------------------------
// TMEM helpers: a CTA of four warps allocates `cols` columns of tensor memory (one warp allocates
// and relinquishes its permit; fences around the barrier), and frees them at the end
template <uint32_t kCols>
__device__ __forceinline__ uint32_t tmem_alloc_cta(uint32_t* holder) {
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(holder))),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  return *holder;
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_free_cta(uint32_t base) {
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "n"(kCols));
}

// kTmem: the column being orthogonalised lives in the thread's TMEM lane instead of shared
// memory, which leaves the whole L1 to the Q columns (the axpy re-reads q_i right after the dot
// product).  Its accesses are warp-collective, so a warp runs the solve if any lane needs it.
// kQCache (with kTmem false): the column in shared memory, and each projected q_i cached in the
// thread's TMEM lane between its dot product and its axpy (TmemQCache); warp-collective as well.
template <class R, bool kTmem, int kThreads, int kMinBlocks, bool kQCache = false, bool kFuse = false,
          bool kHint = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks) lsq_trip(const TrackArgs a) {
  constexpr int L = level<R>::L;
  extern __shared__ double smem[];
  const size_t s = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool in_range = s < a.n_active;
  const SlotInts si{a.si, a.S};
  const int mode = in_range ? si(F_MODE, s) : M_DONE;
  const bool need = mode == M_NEWTON || mode == M_REFINE;
  const int n = a.plan.n;
  const Planar<R> X{a.x, a.S};
  const auto J = PP_WORK(a.J, n * n), Rm = PP_WORK(a.Rm, n * (n + 1) / 2), B = PP_WORK(a.B, n), Y = PP_WORK(a.Y, n);
  if (!kTmem && kQCache) {
    __shared__ uint32_t tmem_holder;
    const uint32_t base = tmem_alloc_cta<128>(&tmem_holder);
    const int warp = threadIdx.x >> 5;
    const TmemQCache<R> qc{base + (static_cast<uint32_t>(32 * (warp & 3)) << 16)};
    const SmemRow<R> C{Planar<R>{smem, blockDim.x}, threadIdx.x};
    // a.lsq_spt slots per thread, one after the other (slot s, s + grid, ...): fewer slots in
    // flight keep more of their Q columns resident in L2 between projections
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (int rep = 0; rep < a.lsq_spt; ++rep) {
      const size_t sr = s + rep * stride;
      const bool in_r = sr < a.n_active;
      const int mode_r = in_r ? si(F_MODE, sr) : M_DONE;
      const bool need_r = mode_r == M_NEWTON || mode_r == M_REFINE;
      if (!__any_sync(0xffffffffu, need_r)) continue;
      const size_t so = in_r ? sr : s;  // out-of-range lanes run on their first slot's scratch
      const bool ok =
          lsq_solve_c<R, decltype(J), SmemRow<R>, true, TmemQCache<R>, kFuse, kHint>(n, n, a.rank_tol, J, Rm, B, Y, so,
                                                                                      C, qc);
      if (need_r) si(F_OK, sr) = ok ? 1 : 0;
      if (need_r && ok) {
        double dxn = 0.0, xn = 0.0;
        for (int v = 0; v < n; ++v) {
          const cx<R> dv = C.ld(v);
          const cx<R> xv = cadd(X.ld(v, sr), dv);
          X.st(v, sr, xv);
          dxn = f_max(dxn, cabsd(dv));
          xn = f_max(xn, cabsd(xv));
        }
        a.sd[D_DXN * a.S + sr] = dxn;
        a.sd[D_XN * a.S + sr] = xn;
      }
    }
    tmem_free_cta<128>(base);
  } else if (!kTmem) {
    if (!need) return;
    const SmemRow<R> C{Planar<R>{smem, blockDim.x}, threadIdx.x};
    const bool ok = lsq_solve_c<R, decltype(J), SmemRow<R>, false>(n, n, a.rank_tol, J, Rm, B, Y, s, C);
    si(F_OK, s) = ok ? 1 : 0;
    if (!ok) return;
    // x += dx; update and iterate norms (tracker.cpp:258-264)
    double dxn = 0.0, xn = 0.0;
    for (int v = 0; v < n; ++v) {
      const cx<R> dv = C.ld(v);
      const cx<R> xv = cadd(X.ld(v, s), dv);
      X.st(v, s, xv);
      dxn = f_max(dxn, cabsd(dv));
      xn = f_max(xn, cabsd(xv));
    }
    a.sd[D_DXN * a.S + s] = dxn;
    a.sd[D_XN * a.S + s] = xn;
  } else {
    __shared__ uint32_t tmem_holder;
    constexpr uint32_t kCols = kThreads == 256 ? 256 : 128;  // two warps per lane quarter at 256 threads
    const uint32_t base = tmem_alloc_cta<kCols>(&tmem_holder);
    const int warp = threadIdx.x >> 5;
    const TmemRow<R> C{base + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + static_cast<uint32_t>((warp >> 2) * n * 4 * L)};
    if (__any_sync(0xffffffffu, need)) {
      const bool ok = lsq_solve_c<R, decltype(J), TmemRow<R>, true>(n, n, a.rank_tol, J, Rm, B, Y, s, C);
      if (need) si(F_OK, s) = ok ? 1 : 0;
      double dxn = 0.0, xn = 0.0;
      for (int v = 0; v < n; ++v) {
        const cx<R> dv = C.ld(v);  // warp-collective
        if (need && ok) {
          const cx<R> xv = cadd(X.ld(v, s), dv);
          X.st(v, s, xv);
          dxn = f_max(dxn, cabsd(dv));
          xn = f_max(xn, cabsd(xv));
        }
      }
      if (need && ok) {
        a.sd[D_DXN * a.S + s] = dxn;
        a.sd[D_XN * a.S + s] = xn;
      }
    }
    tmem_free_cta<kCols>(base);
  }
  (void)L;
}

// ---------------------------------------------------------------------------------------------
// least squares with a compile-time dimension N: the Gram-Schmidt column lives in registers
// ---------------------------------------------------------------------------------------------
// The same operation sequence as lsq_solve_c (linalg.hpp:79-125), with every row loop unrolled so
// the column C is register-resident.  No shared memory is used, so the whole L1 caches the
// solver's Q/R columns.  kHoldQ additionally keeps the projected column q_i in registers (QB)
// from its dot product to its axpy, and refills QB row by row with the next column to be
// projected while the axpy consumes it (software pipelining: the load of row r is issued as soon
// as row r of q_i is dead), so every q_i is read once per projection instead of twice.
template <class R, int N, bool kHoldQ, class GA>
__device__ __forceinline__ bool lsq_solve_reg(double rank_tol, const GA& Q, const GA& Rm, const GA& B,
                                              const GA& Y, size_t s, cx<R> (&C)[N]) {
  const cx<R> zero = czero<R>();
  R max_norm = rfrom<R>(0.0);
#pragma unroll 1
  for (int j = 0; j < N; ++j) {
    R acc = rfrom<R>(0.0);
#pragma unroll
    for (int r = 0; r < N; ++r) acc = radd(acc, cabs2(Q.ld(j * N + r, s)));
    const R nj = rsqrt(acc);
    if (rcmp(nj, max_norm) > 0) max_norm = nj;
  }
  const R tol = rmul(max_norm, rfrom<R>(rank_tol));

  cx<R> QB[kHoldQ ? N : 1];
#pragma unroll 1
  for (int k = 0; k < N; ++k) {
#pragma unroll
    for (int r = 0; r < N; ++r) C[r] = Q.ld(k * N + r, s);
    const int rk = k * (k + 1) / 2;
    if (kHoldQ && k > 0) {
#pragma unroll
      for (int r = 0; r < N; ++r) QB[kHoldQ ? r : 0] = Q.ld(r, s);  // q_0
    }
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
#pragma unroll 1
      for (int i = 0; i < k; ++i) {
        cx<R> rik = zero;
#pragma unroll
        for (int r = 0; r < N; ++r)
          rik = cadd(rik, cmul(cconj(kHoldQ ? QB[kHoldQ ? r : 0] : Q.ld(i * N + r, s)), C[r]));
        const cx<R> prev = pass == 0 ? zero : Rm.ld(i + rk, s);
        Rm.st(i + rk, s, cadd(prev, rik));
        // the next column this thread projects on: q_(i+1), else q_0 of the second pass
        const int nxt = i + 1 < k ? i + 1 : (pass == 0 ? 0 : -1);
#pragma unroll
        for (int r = 0; r < N; ++r) {
          if (kHoldQ) {
            C[r] = csub(C[r], cmul(rik, QB[kHoldQ ? r : 0]));
            if (nxt >= 0) QB[kHoldQ ? r : 0] = Q.ld(nxt * N + r, s);
          } else {
            C[r] = csub(C[r], cmul(rik, Q.ld(i * N + r, s)));
          }
        }
      }
    }
    R acc = rfrom<R>(0.0);
#pragma unroll
    for (int r = 0; r < N; ++r) acc = radd(acc, cabs2(C[r]));
    const R rkk = rsqrt(acc);
    if (rcmp(rkk, tol) <= 0) return false;
    Rm.st(k + rk, s, cx<R>{rkk, rfrom<R>(0.0)});
    const R rinv = rdiv(rfrom<R>(1.0), rkk);
    cx<R> y = zero;
#pragma unroll
    for (int r = 0; r < N; ++r) {
      const cx<R> q = cmulr(C[r], rinv);
      Q.st(k * N + r, s, q);
      y = cadd(y, cmul(cconj(q), B.ld(r, s)));  // y_k = <q_k, b> (linalg.hpp:117)
    }
    Y.st(k, s, y);
  }
  // back substitution R x = y (linalg.hpp:118-122), unrolled so x stays in registers (C)
#pragma unroll
  for (int j = N - 1; j >= 0; --j) {
    cx<R> acc = Y.ld(j, s);
#pragma unroll
    for (int i = j + 1; i < N; ++i) acc = csub(acc, cmul(Rm.ld(j + i * (i + 1) / 2, s), C[i]));
    C[j] = cdiv(acc, Rm.ld(j + j * (j + 1) / 2, s));
  }
  return true;
}

template <class R, int N, bool kHoldQ, int kMinBlocks>
__global__ void __launch_bounds__(128, kMinBlocks) lsq_trip_reg(const TrackArgs a) {
  static_assert(PP_SLOT_TILED, "the register solver reads the slot-tiled solver arrays");
  const size_t s = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= a.n_active) return;
  const SlotInts si{a.si, a.S};
  const int mode = si(F_MODE, s);
  if (mode != M_NEWTON && mode != M_REFINE) return;
  const Tiled<R> J{a.J, static_cast<uint32_t>(N * N)}, Rm{a.Rm, static_cast<uint32_t>(N * (N + 1) / 2)},
      B{a.B, static_cast<uint32_t>(N)}, Y{a.Y, static_cast<uint32_t>(N)};
  cx<R> C[N];
  const bool ok = lsq_solve_reg<R, N, kHoldQ>(a.rank_tol, J, Rm, B, Y, s, C);
  si(F_OK, s) = ok ? 1 : 0;
  if (!ok) return;
  // x += dx; update and iterate norms (tracker.cpp:258-264)
  const Planar<R> X{a.x, a.S};
  double dxn = 0.0, xn = 0.0;
#pragma unroll
  for (int v = 0; v < N; ++v) {
    const cx<R> xv = cadd(X.ld(v, s), C[v]);
    X.st(v, s, xv);
    dxn = f_max(dxn, cabsd(C[v]));
    xn = f_max(xn, cabsd(xv));
  }
  a.sd[D_DXN * a.S + s] = dxn;
  a.sd[D_XN * a.S + s] = xn;
}

// ---------------------------------------------------------------------------------------------
// per-path control: corrector bookkeeping, step control, status, prediction, finalize and record
// output, refill from the start counter.  Shared by the trip kernels (state in SoA global memory)
// and the persistent kernel (state in registers).
// ---------------------------------------------------------------------------------------------
template <class R>
struct SlotState {
  unsigned long long path;
  int mode, it, rit, len, head, consec, corrected, sing, status, reason;
  uint32_t steps, newton, rej;
  R t, h, tnext;
};

// results of the slot's last heavy operation (evaluation, and least-squares update if any)
template <class R>
struct HeavyOut {
  double resid, dxn, xn;
  R resid_r;
  bool ok;
};

// record of start index `path` (inverse of the refill map)
__device__ __forceinline__ size_t record_index(const TrackArgs& a, unsigned long long path) {
  const unsigned long long off = path - a.lo, blk = a.shard_block;
  return static_cast<size_t>(off / (blk * a.shard_n) * blk + off % blk);
}

// X: the slot's working point (xs = its column there); every other per-slot array is global at s
template <class R>
__device__ __forceinline__ void control(const TrackArgs& a, SlotState<R>& st, const HeavyOut<R>& ho,
                                        const Planar<R>& X, size_t xs, size_t s) {
  constexpr int L = level<R>::L;
  if (st.mode == M_DONE) return;
  const int n = a.plan.n;
  const Planar<R> XA{a.xacc, a.S}, HX{a.hx, a.S}, HT{a.ht, a.S};
  const R one = rfrom<R>(1.0);

  // predictor (tracker.cpp:178-214): t_next = min(t + h, 1); Lagrange extrapolation through
  // the accepted history (oldest first), a copy when only the start point is known
  auto predict = [&]() {
    R tn = radd(st.t, st.h);
    if (rcmp(tn, one) >= 0) tn = one;
    st.tnext = tn;
    const int len = st.len, head = st.head;
    if (len == 1) {
      for (int v = 0; v < n; ++v) X.st(v, xs, HX.ld(head * n + v, s));
      return;
    }
    R ts[kHist], w[kHist];
#pragma unroll
    for (int i = 0; i < kHist; ++i)
      if (i < len) ts[i] = HT.ldr((head + i) % kHist, s);
#pragma unroll
    for (int i = 0; i < kHist; ++i) {
      if (i < len) {
        R wi = one;
#pragma unroll
        for (int j = 0; j < kHist; ++j)
          if (j < len && j != i) wi = rmul(wi, rdiv(rsub(tn, ts[j]), rsub(ts[i], ts[j])));
        w[i] = wi;
      }
    }
    for (int v = 0; v < n; ++v) {
      cx<R> acc = czero<R>();
#pragma unroll
      for (int i = 0; i < kHist; ++i)
        if (i < len) acc = cadd(acc, cmulr(HX.ld(((head + i) % kHist) * n + v, s), w[i]));
      X.st(v, xs, acc);
    }
  };

  if (st.mode == M_NEWTON) {
    ++st.it;
    ++st.newton;
    bool done = false;
    if (!ho.ok) {
      st.sing = 1;  // this step failed (tracker.cpp:253-257)
      done = true;
    } else if (ho.resid <= a.rtol && ho.dxn <= f_mul(a.utol, f_max(1.0, ho.xn))) {
      st.corrected = 1;
      done = true;
    } else if (st.it >= a.max_newton) {
      done = true;
    }
    if (done) {
      // step control (tracker.cpp:293-317); history push with FIFO drop at depth 5
      // (tracker.cpp:276-291) kept as a ring buffer
      double xacc_norm = 0.0;
      if (st.corrected) {
        ++st.steps;
        if (st.consec < 255) ++st.consec;
        st.t = st.tnext;
        if (st.len == kHist) {
          st.head = (st.head + 1) % kHist;
          st.len = kHist - 1;
        }
        const int at = (st.head + st.len) % kHist;
        HT.str(at, s, st.tnext);
        for (int v = 0; v < n; ++v) {
          const cx<R> xv = X.ld(v, xs);
          XA.st(v, s, xv);
          HX.st(at * n + v, s, xv);
        }
        ++st.len;
        if (st.consec >= a.expand_after) {
          const R grown = rmuld(st.h, a.expand);
          st.h = rcmp(grown, rfrom<R>(a.h_max)) > 0 ? rfrom<R>(a.h_max) : grown;
        }
        xacc_norm = ho.xn;  // norm of the accepted point = the last iterate's norm
      } else {
        ++st.rej;
        st.consec = 0;
        st.h = rmuld(st.h, a.contract);
        for (int v = 0; v < n; ++v) xacc_norm = f_max(xacc_norm, cabsd(XA.ld(v, s)));
      }
      if (a.ev != nullptr) {
        // the sink's StepEvent (tracker.cpp:312-315): t and h after the decision, this step's
        // corrector iterations, and the status as it stands before this round's check
        const unsigned long long e = atomicAdd(a.ev_count, 1ull);
        if (e < a.ev_cap) {
          StepEventRec r;
          r.path_id = st.path;
          r.t = rtod(st.t);
          r.h = rtod(st.h);
          r.newton_iters = static_cast<uint32_t>(st.it);
          r.status = static_cast<int8_t>(st.status);
          r.accepted = st.corrected ? 1 : 0;
          r.pad[0] = r.pad[1] = 0;
          a.ev[e] = r;
        }
      }
      // status on the accepted point (tracker.cpp:319-338)
      if (xacc_norm > a.div_bound) {
        st.status = ST_FAILED;
        st.reason = RS_DIVERGED;
      } else if (rcmp(st.h, rfrom<R>(a.h_min)) < 0) {
        st.status = ST_FAILED;
        st.reason = st.sing ? RS_SINGULAR : RS_UNDERFLOW;
      } else if (st.steps > a.max_steps) {
        st.status = ST_FAILED;
        st.reason = RS_MAXSTEPS;
      } else if (rcmp(st.t, one) == 0 && st.corrected) {
        st.status = ST_SUCCESS;
      }

      if (st.status == ST_ACTIVE) {
        predict();
        st.it = 0;
        st.corrected = 0;
        st.sing = 0;
      } else {
        const size_t rec = record_index(a, st.path);
        uint8_t flag = 0;
        if (st.status == ST_FAILED && st.reason != RS_DIVERGED && f_sub(1.0, rtod(st.t)) < 0.01 && st.len >= 3) {
          // terminal divergence test inputs (tracker.cpp:406-432); the log ratio is taken on
          // the host with the reference's libm
          double first = 0.0, prev = -1.0, last = 0.0;
          bool growing = true;
          for (int i = 0; i < st.len; ++i) {
            double nrm = 0.0;
            const int at = (st.head + i) % kHist;
            for (int v = 0; v < n; ++v) nrm = f_max(nrm, cabsd(HX.ld(at * n + v, s)));
            if (nrm <= prev) growing = false;
            if (i == 0) first = nrm;
            prev = nrm;
            last = nrm;
          }
          const double uf = f_sub(1.0, rtod(HT.ldr(st.head, s)));
          const double ul = f_sub(1.0, rtod(HT.ldr((st.head + st.len - 1) % kHist, s)));
          if (growing && first > 0.0 && ul > 0.0 && uf > ul) {
            flag = 1;
            a.rec_div[rec * 4 + 0] = first;
            a.rec_div[rec * 4 + 1] = last;
            a.rec_div[rec * 4 + 2] = uf;
            a.rec_div[rec * 4 + 3] = ul;
          }
        }
        a.rec_divflag[rec] = flag;
        if (st.status == ST_SUCCESS) {
          st.mode = M_REFINE;  // x == xacc here
          st.rit = 0;
        } else {
          for (int v = 0; v < n; ++v) X.st(v, xs, XA.ld(v, s));
          st.mode = M_FINAL;
        }
      }
    }
  } else if (st.mode == M_REFINE) {
    // endpoint refinement at t = 1: at most 3 iterations, stopping on the update test alone
    // or on a failed solve (tracker.cpp:446-478); the refined point becomes xacc
    ++st.rit;
    const bool stop = !ho.ok || ho.dxn <= f_mul(a.utol, f_max(1.0, ho.xn));
    if (stop || st.rit >= 3) st.mode = M_FINAL;
  } else if (st.mode == M_FINAL) {
    // final residual ||f(xacc)|| at level R and the certificate (tracker.cpp:480-506)
    const size_t rec = record_index(a, st.path);
    int st_out = st.status, rs_out = st.reason;
    if (st_out == ST_SUCCESS && rtod(ho.resid_r) > f_mul(10.0, a.rtol)) {
      st_out = ST_FAILED;
      rs_out = RS_NOCERT;
    }
    for (int v = 0; v < n; ++v) st_flat<R>(a.rec_x + (rec * n + v) * 2 * L, X.ld(v, xs));
#pragma unroll
    for (int l = 0; l < L; ++l) a.rec_res[rec * L + l] = level<R>::get(ho.resid_r, l);
    a.rec_status[rec] = static_cast<int8_t>(st_out);
    a.rec_reason[rec] = static_cast<uint8_t>(rs_out);
    a.rec_steps[rec] = st.steps;
    a.rec_newton[rec] = st.newton;
    a.rec_rej[rec] = st.rej;
    st.mode = M_IDLE;
  }

  if (st.mode == M_IDLE) {
    // refill: next start index; seed (tracker.cpp:135-153) and the first prediction
    const unsigned long long k = atomicAdd(a.next, 1ull);
    if (k >= a.count) {
      st.mode = M_DONE;
    } else {
      const unsigned long long blk = a.shard_block;
      st.path = a.lo + ((k / blk) * a.shard_n + a.shard_r) * blk + k % blk;
      if (a.total_degree) {
        unsigned long long rem = st.path;
        for (int i = n - 1; i >= 0; --i) {
          const uint32_t d = __ldg(a.degrees + i);
          const unsigned long long q = rem / d;
          const uint32_t ri = static_cast<uint32_t>(rem - q * d);
          rem = q;
          X.st(i, xs, ld_flat<R>(a.roots + (static_cast<size_t>(__ldg(a.root_off + i)) + ri) * 2 * L));
        }
      } else {
        for (int v = 0; v < n; ++v)
          X.st(v, xs, ld_flat<R>(a.explicit_x + (static_cast<size_t>(st.path - a.lo) * n + v) * 2 * L));
      }
      st.head = 0;
      st.len = 1;
      HT.str(0, s, rfrom<R>(0.0));
      for (int v = 0; v < n; ++v) {
        const cx<R> xv = X.ld(v, xs);
        XA.st(v, s, xv);
        HX.st(v, s, xv);
      }
      st.t = rfrom<R>(0.0);
      st.h = rfrom<R>(a.h_init);
      st.steps = st.newton = st.rej = 0;
      st.consec = 0;
      st.status = ST_ACTIVE;
      st.reason = RS_NONE;
      predict();
      st.mode = M_NEWTON;
      st.it = 0;
      st.corrected = 0;
      st.sing = 0;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// one control step of slot s with its state in the SoA global arrays; returns the new mode
// ---------------------------------------------------------------------------------------------
template <class R>
__device__ __forceinline__ int step_slot(const TrackArgs& a, size_t s, const Planar<R>& X, size_t xs,
                                         const HeavyOut<R>& ho) {
  const SlotInts si{a.si, a.S};
  const Planar<R> SR{a.sr, a.S};
  SlotState<R> st;
  st.mode = si(F_MODE, s);
  if (st.mode == M_DONE) return M_DONE;
  st.path = a.spath[s];
  st.it = si(F_IT, s);
  st.rit = si(F_RIT, s);
  st.len = si(F_LEN, s);
  st.head = si(F_HEAD, s);
  st.consec = si(F_CONSEC, s);
  st.corrected = si(F_CORR, s);
  st.sing = si(F_SING, s);
  st.status = si(F_STATUS, s);
  st.reason = si(F_REASON, s);
  st.steps = si(F_STEPS, s);
  st.newton = si(F_NEWTON, s);
  st.rej = si(F_REJ, s);
  st.t = SR.ldr(R_T, s);
  st.h = SR.ldr(R_H, s);
  st.tnext = SR.ldr(R_TNEXT, s);
  control<R>(a, st, ho, X, xs, s);
  a.spath[s] = st.path;
  si(F_MODE, s) = st.mode;
  si(F_IT, s) = st.it;
  si(F_RIT, s) = st.rit;
  si(F_LEN, s) = st.len;
  si(F_HEAD, s) = st.head;
  si(F_CONSEC, s) = st.consec;
  si(F_CORR, s) = st.corrected;
  si(F_SING, s) = st.sing;
  si(F_STATUS, s) = st.status;
  si(F_REASON, s) = st.reason;
  si(F_STEPS, s) = static_cast<int32_t>(st.steps);
  si(F_NEWTON, s) = static_cast<int32_t>(st.newton);
  si(F_REJ, s) = static_cast<int32_t>(st.rej);
  SR.str(R_T, s, st.t);
  SR.str(R_H, s, st.h);
  SR.str(R_TNEXT, s, st.tnext);
  return st.mode;
}

// ---------------------------------------------------------------------------------------------
// control kernel of tail mode (thread per slot; the thread-per-path trips fuse it into
// ctrl_eval_trip)
// ---------------------------------------------------------------------------------------------
template <class R>
__global__ void __launch_bounds__(128) step_trip(const TrackArgs a, unsigned* busy_out) {
  const size_t s = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool in_range = s < a.n_active;
  int mode = M_DONE;
  if (in_range) {
    const SlotInts si{a.si, a.S};
    const Planar<R> X{a.x, a.S}, SR{a.sr, a.S};
    HeavyOut<R> ho;
    ho.ok = si(F_OK, s) != 0;
    ho.resid = a.sd[D_RESID * a.S + s];
    ho.dxn = a.sd[D_DXN * a.S + s];
    ho.xn = a.sd[D_XN * a.S + s];
    ho.resid_r = SR.ldr(R_RESID, s);
    mode = step_slot<R>(a, s, X, s, ho);
  }
  // every busy slot has exactly one heavy operation pending for the next trip
  const unsigned busy = __ballot_sync(0xffffffffu, in_range && mode != M_DONE);
  const unsigned solve = __ballot_sync(0xffffffffu, in_range && (mode == M_NEWTON || mode == M_REFINE));
  if ((threadIdx.x & 31) == 0 && busy != 0) {
    atomicAdd(busy_out, static_cast<unsigned>(__popc(busy)));
    atomicAdd(a.work, static_cast<unsigned long long>(__popc(busy)));
    atomicAdd(a.work + 1, static_cast<unsigned long long>(__popc(solve)));
  }
}

// ---------------------------------------------------------------------------------------------
// trip kernel 1 (thread per path): control, then the evaluation of H and dH/dx at the slot's
// point.  The point is staged in shared memory, the control step (step control, predictor,
// finalize, refill; tracker.cpp:178-338, 402-509) updates it there, the evaluation reads it, and
// it is written back for the least-squares kernel.  The control part counts the slots with work
// in this trip (busy_out) and the evaluations / solves issued (a.work).
// ---------------------------------------------------------------------------------------------
// kStage: the plan tables (term info, positions, base factors, coefficients) are copied into
// shared memory by one bulk TMA transfer each (cp.async.bulk, completion on an mbarrier) when the
// CTA starts, and the evaluation reads them from there (PlanArgs::stage_* give the layout)
template <class R, int KMAX, bool kTmem, int kMinBlocks, bool kStage = false>
__global__ void __launch_bounds__(128, kMinBlocks) ctrl_eval_trip(const TrackArgs a, unsigned* busy_out) {
  constexpr int L = level<R>::L;
  extern __shared__ double smem[];
  PlanArgs pa_s = a.plan;
  if constexpr (kStage) {
    __shared__ __align__(8) unsigned long long mbar;
    char* tab = reinterpret_cast<char*>(smem) + a.plan.stage_offset;
    const uint32_t mb = static_cast<uint32_t>(__cvta_generic_to_shared(&mbar));
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(a.plan.stage_bytes[4])
                   : "memory");
      const void* src[4] = {a.plan.term_info, a.plan.pos, a.plan.base, a.plan.coeff};
      uint32_t off = 0;
      for (int q = 0; q < 4; ++q) {
        if (a.plan.stage_bytes[q] != 0)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                           static_cast<uint32_t>(__cvta_generic_to_shared(tab + off))),
                       "l"(src[q]), "r"(a.plan.stage_bytes[q]), "r"(mb)
                       : "memory");
        off += a.plan.stage_bytes[q];
      }
    }
    __syncthreads();
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.b32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(mb) : "memory");
    pa_s.term_info = reinterpret_cast<const int32_t*>(tab);
    pa_s.pos = reinterpret_cast<const uint32_t*>(tab + a.plan.stage_bytes[0]);
    pa_s.base = reinterpret_cast<const uint32_t*>(tab + a.plan.stage_bytes[0] + a.plan.stage_bytes[1]);
    pa_s.coeff = reinterpret_cast<const double*>(tab + a.plan.stage_bytes[0] + a.plan.stage_bytes[1] +
                                                 a.plan.stage_bytes[2]);
  }
  const size_t s = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool in_range = s < a.n_active;
  const int n = a.plan.n;
  const size_t ls = threadIdx.x;
  const Planar<R> XS{smem, blockDim.x};
  // TMEM variant: the CTA's open rows live in tensor memory (warp w: lanes 32*(w%4) .. +31,
  // columns (w/4) * n*4L ..); one warp allocates, all fence around the barrier
  __shared__ uint32_t tmem_base;
  const uint32_t kCols = a.tmem_cols;  // power of two >= n*4L, chosen by the host
  if (kTmem) {
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base))),
                   "r"(kCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
  }
  const int warp = threadIdx.x >> 5;
  const uint32_t row_base = kTmem ? tmem_base + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                                        static_cast<uint32_t>((warp >> 2) * n * 4 * L)
                                  : 0u;
  int mode = M_DONE;
  bool need = false;
  R t = rfrom<R>(1.0);
  if (in_range) {
    const SlotInts si{a.si, a.S};
    mode = si(F_MODE, s);
    if (mode != M_DONE) {
      const Planar<R> X{a.x, a.S}, SR{a.sr, a.S};
      for (int v = 0; v < n; ++v) XS.st(v, ls, X.ld(v, s));
      HeavyOut<R> ho;
      ho.ok = si(F_OK, s) != 0;
      ho.resid = a.sd[D_RESID * a.S + s];
      ho.dxn = a.sd[D_DXN * a.S + s];
      ho.xn = a.sd[D_XN * a.S + s];
      ho.resid_r = SR.ldr(R_RESID, s);
      mode = step_slot<R>(a, s, XS, ls, ho);
      need = mode == M_NEWTON || mode == M_REFINE || mode == M_FINAL;
      if (mode == M_NEWTON) t = SR.ldr(R_TNEXT, s);
    }
  }
  const auto J = PP_WORK(a.J, n * a.plan.n_polys), B = PP_WORK(a.B, a.plan.n_polys);
  double resid;
  R resid_r;
  if (kTmem) {
    // warp-collective TMEM accesses: the warp evaluates if any lane needs it; the other lanes
    // run the same plan on their (unused) point and discard the results
    if (__any_sync(0xffffffffu, need)) {
      eval_hj<R, KMAX, kStage>(pa_s, XS, TmemRow<R>{row_base}, ls, t, B, J, s, resid, resid_r);
    }
  } else if (need) {
    const Planar<R> JR{smem + static_cast<size_t>(n) * 2 * L * blockDim.x, blockDim.x};
    eval_hj<R, KMAX, kStage>(pa_s, XS, SmemRow<R>{JR, ls}, ls, t, B, J, s, resid, resid_r);
  }
  if (need) {
    const Planar<R> X{a.x, a.S}, SR{a.sr, a.S};
    a.sd[D_RESID * a.S + s] = resid;
    SR.str(R_RESID, s, resid_r);
    for (int v = 0; v < n; ++v) X.st(v, s, XS.ld(v, ls));
  }
  const unsigned busy = __ballot_sync(0xffffffffu, in_range && mode != M_DONE);
  const unsigned solve = __ballot_sync(0xffffffffu, in_range && (mode == M_NEWTON || mode == M_REFINE));
  if ((threadIdx.x & 31) == 0 && busy != 0) {
    atomicAdd(busy_out, static_cast<unsigned>(__popc(busy)));
    atomicAdd(a.work, static_cast<unsigned long long>(__popc(busy)));
    atomicAdd(a.work + 1, static_cast<unsigned long long>(__popc(solve)));
  }
  if (kTmem) {
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (threadIdx.x < 32)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(kCols));
  }
}

// ---------------------------------------------------------------------------------------------
// tail mode: one warp per path slot
// ---------------------------------------------------------------------------------------------
// When only a few paths remain (after compaction), a thread per path leaves the GPU idle and each
// trip costs a lone warp's issue time.  These kernels give each remaining path a whole warp and
// split its trip across the lanes while keeping the reference's operation order, so results are
// bitwise those of the thread-per-path kernels:
//  * evaluation: lanes compute the terms' products independently into contribution slots; each
//    accumulator (H_p, dH_p/dx_v) then sums its slots in plan order (build_accumulation_lists);
//  * least squares: lanes own the rows of the Gram-Schmidt column operations (products, axpy,
//    scaling); every sequential sum of the reference (dot products, norms, back substitution)
//    is carried out in order by lane 0.

// lane group of the tail-mode kernels: G consecutive lanes serve one path slot, 32 / G slots per warp
template <int G>
struct LaneGroup {
  static constexpr int kPerWarp = 32 / G;
  int gl;         // lane within the group
  int first;      // the group's first lane in the warp
  unsigned mask;  // the group's lanes
  __device__ __forceinline__ LaneGroup() {
    const int lane = threadIdx.x & 31;
    gl = lane % G;
    first = lane - gl;
    mask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << first);
  }
  __device__ __forceinline__ size_t slot() const {
    return (static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kPerWarp + first / G;
  }
  __device__ __forceinline__ int index_in_block() const { return (threadIdx.x >> 5) * kPerWarp + first / G; }
  __device__ __forceinline__ void sync() const { __syncwarp(mask); }
  // max over the group (rcmp order; equal values are identical, so the result is exact)
  template <class R>
  __device__ __forceinline__ R rmax(R v) const {
    constexpr int L = level<R>::L;
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
      R o;
#pragma unroll
      for (int l = 0; l < L; ++l) level<R>::set(o, l, __shfl_xor_sync(mask, level<R>::get(v, l), off));
      if (rcmp(o, v) > 0) v = o;
    }
    return v;
  }
  __device__ __forceinline__ double fmax(double v) const {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) v = f_max(v, __shfl_xor_sync(mask, v, off));
    return v;
  }
  template <class R>
  __device__ __forceinline__ R bcast(R v) const {  // the group's first lane's value
    constexpr int L = level<R>::L;
#pragma unroll
    for (int l = 0; l < L; ++l) level<R>::set(v, l, __shfl_sync(mask, level<R>::get(v, l), first));
    return v;
  }
};

// G lanes per path slot (G = 32: a warp per path)
template <class R, int KMAX, int G>
__global__ void __launch_bounds__(128) eval_coop(const TrackArgs a) {
  constexpr int L = level<R>::L;
  extern __shared__ double smem[];
  const LaneGroup<G> g;
  const int lane = g.gl;
  const size_t s = g.slot();
  if (s >= a.n_active) return;  // group-uniform
  const SlotInts si{a.si, a.S};
  const int mode = si(F_MODE, s);
  if (mode != M_NEWTON && mode != M_REFINE && mode != M_FINAL) return;
  const PlanArgs& pa = a.plan;
  const int n = pa.n, np = pa.n_polys;
  const size_t per_slot = static_cast<size_t>(n + pa.n_slots) * 2 * L;
  double* base = smem + static_cast<size_t>(g.index_in_block()) * per_slot;
  const Planar<R> XS{base, 1}, SL{base + static_cast<size_t>(n) * 2 * L, 1};
  const Planar<R> X{a.x, a.S}, SR{a.sr, a.S};
  const auto J = PP_WORK(a.J, n * np), B = PP_WORK(a.B, np);
  for (int v = lane; v < n; v += G) XS.st(v, 0, X.ld(v, s));
  g.sync();
  const R t = mode == M_NEWTON ? SR.ldr(R_TNEXT, s) : rfrom<R>(1.0);
  const R u = rsub(rfrom<R>(1.0), t);
  for (int i = lane; i < pa.n_terms; i += G) {
    const int slot = static_cast<int>(__ldg(pa.term_slot + i));
    int poly;
    eval_term<R, KMAX>(
        pa, i, XS, 0, t, u, poly, [&](const cx<R>& v) { SL.st(slot, 0, v); },
        [&](int j, int, const cx<R>& w) { SL.st(slot + 1 + j, 0, w); }, [&](int) {});
  }
  g.sync();
  double resid = 0.0;
  R resid_r = rfrom<R>(0.0);
  const int n_acc = np + np * n;
  for (int acc = lane; acc < n_acc; acc += G) {
    cx<R> sum = czero<R>();
    const int e = static_cast<int>(__ldg(pa.acc_off + acc + 1));
    for (int q = static_cast<int>(__ldg(pa.acc_off + acc)); q < e; ++q)
      sum = cadd(sum, SL.ld(static_cast<int>(__ldg(pa.acc_idx + q)), 0));
    if (acc < np) {
      B.st(acc, s, cneg(sum));
      const R m = cabsr(sum);
      resid = f_max(resid, rtod(m));
      if (rcmp(m, resid_r) > 0) resid_r = m;
    } else {
      const int p = (acc - np) / n, v = (acc - np) - p * n;
      J.st(v * np + p, s, sum);
    }
  }
  resid = g.fmax(resid);
  resid_r = g.template rmax<R>(resid_r);
  if (lane == 0) {
    a.sd[D_RESID * a.S + s] = resid;
    SR.str(R_RESID, s, resid_r);
  }
}

// matrix access for the warp-per-path solve: the path's Q and R either staged in shared memory
// (small n) or left in the slot-tiled global arrays (large n, where a shared-memory copy would
// leave room for one or two warps per SM)
template <class R>
struct CoopMat {
  Planar<R> sm;  // shared memory copy (stride 1), used when tiled.base == nullptr
  Tiled<R> tiled;
  size_t s;
  __device__ __forceinline__ cx<R> ld(int e) const { return tiled.base ? tiled.ld(e, s) : sm.ld(e, 0); }
  __device__ __forceinline__ void st(int e, const cx<R>& v) const {
    if (tiled.base) tiled.st(e, s, v);
    else sm.st(e, 0, v);
  }
};

// Warp-per-path least squares, right-looking: as soon as q_k is final, every later column j
// receives its first-pass projection on q_k (one lane per column, rows in order); column k's own
// second pass then runs row-parallel with the sums in order on lanes 0/1.  Each column still
// sees q_0, q_1, ... in the reference's order in both passes (linalg.hpp:88-100), so the result is
// bitwise that of lsq_solve_c, with the first pass off the critical path.
template <class R, bool kGlobalQ, int G>
__global__ void __launch_bounds__(128) lsq_coop(const TrackArgs a) {
  constexpr int L = level<R>::L;
  extern __shared__ double smem[];
  const LaneGroup<G> g;
  const int lane = g.gl;
  const size_t s = g.slot();
  if (s >= a.n_active) return;  // group-uniform
  const SlotInts si{a.si, a.S};
  const int mode = si(F_MODE, s);
  if (mode != M_NEWTON && mode != M_REFINE) return;
  const int n = a.plan.n;
  const int nR = n * (n + 1) / 2;
  // per warp in shared memory: b, y, x (the update), row products P [, Q (n*n), R (packed)]
  const size_t per_warp = static_cast<size_t>(4 * n + (kGlobalQ ? 0 : n * n + nR)) * 2 * L;
  double* base = smem + static_cast<size_t>(g.index_in_block()) * per_warp;
  const Planar<R> BS{base, 1}, YS{base + n * 2 * L, 1}, DS{base + 2 * n * 2 * L, 1}, PS{base + 3 * n * 2 * L, 1};
  const Planar<R> X{a.x, a.S};
  const auto J = PP_WORK(a.J, n * n), B = PP_WORK(a.B, n);
  CoopMat<R> Q, RM;
  Q.s = RM.s = s;
  if (kGlobalQ) {
    // the evaluation wrote J through PP_WORK: the global-Q solver reads the same slot-tiled layout
    static_assert(PP_SLOT_TILED, "lsq_coop<R, true> reads the slot-tiled solver arrays");
    Q.tiled = Tiled<R>{a.J, static_cast<uint32_t>(n * n)};
    RM.tiled = Tiled<R>{a.Rm, static_cast<uint32_t>(nR)};
  } else {
    Q.tiled.base = RM.tiled.base = nullptr;
    Q.sm = Planar<R>{base + 4 * n * 2 * L, 1};
    RM.sm = Planar<R>{base + (4 * n + n * n) * 2 * L, 1};
    for (int e = lane; e < n * n; e += G) Q.st(e, J.ld(e, s));
  }
  for (int e = lane; e < n; e += G) BS.st(e, 0, B.ld(e, s));
  g.sync();
  const cx<R> zero = czero<R>();

  // column norms (col_norm, linalg.hpp:57-66): one column per lane, rows in order
  R max_norm = rfrom<R>(0.0);
  for (int j = lane; j < n; j += G) {
    R acc = rfrom<R>(0.0);
    for (int r = 0; r < n; ++r) acc = radd(acc, cabs2(Q.ld(j * n + r)));
    const R nj = rsqrt(acc);
    if (rcmp(nj, max_norm) > 0) max_norm = nj;
  }
  max_norm = g.template rmax<R>(max_norm);
  const R tol = rmul(max_norm, rfrom<R>(a.rank_tol));

  bool ok = true;
  for (int k = 0; k < n; ++k) {
    const int rk = k * (k + 1) / 2;
    // second pass of column k (its first pass arrived from the right-looking steps below)
    for (int i = 0; i < k; ++i) {
      for (int r = lane; r < n; r += G) PS.st(r, 0, cmul(cconj(Q.ld(i * n + r)), Q.ld(k * n + r)));
      g.sync();
      if (lane < 2) {  // dot_conj: rows in order (linalg.hpp:69-73); lane 0 real, lane 1 imaginary part
        R acc = rfrom<R>(0.0);
        for (int r = 0; r < n; ++r) acc = radd(acc, PS.ldr(2 * r + lane, 0));
        __syncwarp(g.mask & (0x3u << g.first));
        PS.str(lane, 0, acc);
      }
      g.sync();
      const cx<R> rik = PS.ld(0, 0);
      if (lane == 0) RM.st(i + rk, cadd(RM.ld(i + rk), rik));  // R(i,k) += rik (second pass)
      g.sync();
      for (int r = lane; r < n; r += G) Q.st(k * n + r, csub(Q.ld(k * n + r), cmul(rik, Q.ld(i * n + r))));
      g.sync();
    }
    for (int r = lane; r < n; r += G) {
      const R v = cabs2(Q.ld(k * n + r));
      PS.st(r, 0, cx<R>{v, rfrom<R>(0.0)});
    }
    g.sync();
    R rkk = rfrom<R>(0.0);
    if (lane == 0) {
      R acc = rfrom<R>(0.0);
      for (int r = 0; r < n; ++r) acc = radd(acc, PS.ld(r, 0).re);
      rkk = rsqrt(acc);
    }
    rkk = g.template bcast<R>(rkk);
    g.sync();
    if (rcmp(rkk, tol) <= 0) {
      ok = false;
      break;
    }
    const R rinv = rdiv(rfrom<R>(1.0), rkk);  // every lane computes the same value
    if (lane == 0) RM.st(k + rk, cx<R>{rkk, rfrom<R>(0.0)});
    for (int r = lane; r < n; r += G) {
      const cx<R> q = cmulr(Q.ld(k * n + r), rinv);
      Q.st(k * n + r, q);
      PS.st(r, 0, cmul(cconj(q), BS.ld(r, 0)));
    }
    g.sync();
    if (lane < 2) {  // y_k = <q_k, b> (linalg.hpp:117), real / imaginary part
      R y = rfrom<R>(0.0);
      for (int r = 0; r < n; ++r) y = radd(y, PS.ldr(2 * r + lane, 0));
      YS.str(2 * k + lane, 0, y);
    }
    // right-looking first pass: q_k projected out of every later column, one lane per column
    // (R(k,j) = 0 + r as the reference's out.r.at(i, k) += rik on a zero matrix)
    for (int j = k + 1 + lane; j < n; j += G) {
      cx<R> r = zero;
      for (int row = 0; row < n; ++row) r = cadd(r, cmul(cconj(Q.ld(k * n + row)), Q.ld(j * n + row)));
      RM.st(k + j * (j + 1) / 2, cadd(zero, r));
      for (int row = 0; row < n; ++row) Q.st(j * n + row, csub(Q.ld(j * n + row), cmul(r, Q.ld(k * n + row))));
    }
    g.sync();
  }
  if (lane == 0) si(F_OK, s) = ok ? 1 : 0;
  if (!ok) return;
  // back substitution R x = y (linalg.hpp:118-122): products by the lanes, sums in order by lanes 0/1
  for (int j = n - 1; j >= 0; --j) {
    for (int i = j + 1 + lane; i < n; i += G) PS.st(i, 0, cmul(RM.ld(j + i * (i + 1) / 2), DS.ld(i, 0)));
    g.sync();
    if (lane < 2) {  // real / imaginary part of acc -= R_ji x_i, in order
      R acc = YS.ldr(2 * j + lane, 0);
      for (int i = j + 1; i < n; ++i) acc = rsub(acc, PS.ldr(2 * i + lane, 0));
      PS.str(lane, 0, acc);
    }
    g.sync();
    if (lane == 0) DS.st(j, 0, cdiv(PS.ld(0, 0), RM.ld(j + j * (j + 1) / 2)));
    g.sync();
  }
  // x += dx; update and iterate norms (tracker.cpp:258-264)
  double dxn = 0.0, xn = 0.0;
  for (int v = lane; v < n; v += G) {
    const cx<R> dv = DS.ld(v, 0);
    const cx<R> xv = cadd(X.ld(v, s), dv);
    X.st(v, s, xv);
    dxn = f_max(dxn, cabsd(dv));
    xn = f_max(xn, cabsd(xv));
  }
  dxn = g.fmax(dxn);
  xn = g.fmax(xn);
  if (lane == 0) {
    a.sd[D_DXN * a.S + s] = dxn;
    a.sd[D_XN * a.S + s] = xn;
  }
}

// ---------------------------------------------------------------------------------------------
// kernel-level parity entry points
// ---------------------------------------------------------------------------------------------
template <class R, int KMAX>
__global__ void __launch_bounds__(128) eval_kernel(const EvalArgs a) {
  constexpr int L = level<R>::L;
  extern __shared__ double smem[];
  const size_t s = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= a.batch) return;
  const int n = a.plan.n;
  const size_t ls = threadIdx.x;
  const Planar<R> X{smem, blockDim.x};
  const Planar<R> JR{smem + static_cast<size_t>(n) * 2 * L * blockDim.x, blockDim.x};
  const Planar<R> XG{const_cast<double*>(a.x), a.batch}, TG{const_cast<double*>(a.t), a.batch};
  for (int v = 0; v < n; ++v) X.st(v, ls, XG.ld(v, s));
  const R t = TG.ldr(0, s);
  const Planar<R> B{a.sys, a.batch}, J{a.jac, a.batch};
  double rd;
  R rr;
  eval_hj<R, KMAX>(a.plan, X, SmemRow<R>{JR, ls}, ls, t, B, J, s, rd, rr);
  // B holds -H; return H
  for (int p = 0; p < a.plan.n_polys; ++p) B.st(p, s, cneg(B.ld(p, s)));
}

// The corrector alone (PathBatch::newton_correct after set_prediction, tracker.cpp:216-274 and
// tracker.hpp:135-136): each thread runs up to max_newton Newton iterations at its own (t, x):
// evaluation, least squares, x += dx, the residual / update test -- the same operations the
// tracker's corrector performs -- and reports the iterations, the convergence and singularity
// flags and the final iterate.  Shared memory per thread: the point, the open Jacobian row and the
// Gram-Schmidt column.
template <class R, int KMAX>
__global__ void __launch_bounds__(128) newton_kernel(const NewtonArgs a) {
  constexpr int L = level<R>::L;
  extern __shared__ double smem[];
  const size_t s = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= a.batch) return;
  const int n = a.plan.n;
  const size_t ls = threadIdx.x, col = static_cast<size_t>(n) * 2 * L * blockDim.x;
  const Planar<R> XS{smem, blockDim.x}, JR{smem + col, blockDim.x};
  const SmemRow<R> C{Planar<R>{smem + 2 * col, blockDim.x}, ls};
  const Planar<R> XG{a.x, a.batch}, TG{const_cast<double*>(a.t), a.batch};
  const Planar<R> J{a.J, a.batch}, Rm{a.Rm, a.batch}, B{a.B, a.batch}, Y{a.Y, a.batch};
  for (int v = 0; v < n; ++v) XS.st(v, ls, XG.ld(v, s));
  const R t = TG.ldr(0, s);
  uint32_t iters = 0;
  uint8_t corrected = 0, sing = 0;
  for (int it = 0; it < a.max_newton; ++it) {
    ++iters;
    double resid;
    R resid_r;
    eval_hj<R, KMAX>(a.plan, XS, SmemRow<R>{JR, ls}, ls, t, B, J, s, resid, resid_r);
    if (!lsq_solve_c<R, Planar<R>, SmemRow<R>, false>(n, n, a.rank_tol, J, Rm, B, Y, s, C)) {
      sing = 1;
      break;
    }
    double dxn = 0.0, xn = 0.0;
    for (int v = 0; v < n; ++v) {
      const cx<R> dv = C.ld(v);
      const cx<R> xv = cadd(XS.ld(v, ls), dv);
      XS.st(v, ls, xv);
      dxn = f_max(dxn, cabsd(dv));
      xn = f_max(xn, cabsd(xv));
    }
    if (resid <= a.rtol && dxn <= f_mul(a.utol, f_max(1.0, xn))) {
      corrected = 1;
      break;
    }
  }
  for (int v = 0; v < n; ++v) XG.st(v, s, XS.ld(v, ls));
  a.iters[s] = iters;
  a.corrected[s] = corrected;
  a.singular[s] = sing;
}

template <class R>
__global__ void __launch_bounds__(128) lsq_kernel(const LsqArgs a) {
  extern __shared__ double smem[];
  const size_t s = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= a.batch) return;
  const Planar<R> Q{a.a, a.batch}, Rm{a.r, a.batch}, B{a.b, a.batch}, Y{a.y, a.batch}, X{a.x, a.batch};
  const Planar<R> C{smem, blockDim.x};
  const bool ok = lsq_solve_c<R, Planar<R>, SmemRow<R>, false>(a.n, a.m, a.rank_tol, Q, Rm, B, Y, s, SmemRow<R>{C, threadIdx.x});
  a.ok[s] = ok ? 1 : 0;
  for (int v = 0; v < a.n; ++v) X.st(v, s, ok ? C.ld(v, threadIdx.x) : czero<R>());
}

}  // namespace dev
}  // namespace pp

// instantiate the kernels of one (level, KMAX) variant; KMAX bounds the distinct variables of a
// monomial (the length of the Speelpenning prefix stack)
#define PP_VARIANT(R, KM)                                                             \
  {KM, reinterpret_cast<const void*>(&pp::dev::ctrl_eval_trip<R, KM, false, PP_EVAL_MINB>),                     \
   reinterpret_cast<const void*>(&pp::dev::lsq_trip<R, false, 128, PP_LSQ_MINB>),                              \
   reinterpret_cast<const void*>(&pp::dev::step_trip<R>),                             \
   reinterpret_cast<const void*>(&pp::dev::eval_kernel<R, KM>),                       \
   reinterpret_cast<const void*>(&pp::dev::lsq_kernel<R>),                            \
   {reinterpret_cast<const void*>(&pp::dev::eval_coop<R, KM, 32>),                    \
    reinterpret_cast<const void*>(&pp::dev::eval_coop<R, KM, 8>),                     \
    reinterpret_cast<const void*>(&pp::dev::eval_coop<R, KM, 4>)},                    \
   {reinterpret_cast<const void*>(&pp::dev::lsq_coop<R, false, 32>),                  \
    reinterpret_cast<const void*>(&pp::dev::lsq_coop<R, false, 8>),                   \
    reinterpret_cast<const void*>(&pp::dev::lsq_coop<R, false, 4>)},                  \
   {reinterpret_cast<const void*>(&pp::dev::lsq_coop<R, true, 32>),                   \
    reinterpret_cast<const void*>(&pp::dev::lsq_coop<R, true, 8>),                    \
    reinterpret_cast<const void*>(&pp::dev::lsq_coop<R, true, 4>)},                   \
   reinterpret_cast<const void*>(&pp::dev::ctrl_eval_trip<R, KM, true, (sizeof(R) < 32 ? 4 : 1)>),             \
   reinterpret_cast<const void*>(&pp::dev::lsq_trip<R, true, 256, 2>),                                        \
   reinterpret_cast<const void*>(&pp::dev::lsq_trip<R, false, 128, PP_LSQ_MINB, true>),                        \
   reinterpret_cast<const void*>(&pp::dev::lsq_trip<R, false, 128, PP_LSQ_MINB, true, true>),                  \
   reinterpret_cast<const void*>(&pp::dev::newton_kernel<R, KM>),                                              \
   reinterpret_cast<const void*>(&pp::dev::ctrl_eval_trip<R, KM, true, (sizeof(R) < 32 ? 4 : 1), true>),          \
   reinterpret_cast<const void*>(&pp::dev::lsq_trip<R, false, 128, PP_LSQ_MINB, true, true, true>)}

// register-resident least-squares solvers of one level for dimension N
#define PP_LSQ_REG(R, N)                                                                        \
  {N, reinterpret_cast<const void*>(&pp::dev::lsq_trip_reg<R, N, false, 4>),                   \
   reinterpret_cast<const void*>(&pp::dev::lsq_trip_reg<R, N, true, (sizeof(R) == 8 ? 4 : 2)>)}
