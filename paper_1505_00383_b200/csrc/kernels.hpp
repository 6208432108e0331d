// kernels.hpp -- argument blocks and the registry of compiled kernel variants.
//
// Kernels are templated on the level R (double / dd / qd) and KMAX (largest number of distinct
// variables in a monomial, i.e. the length of the Speelpenning prefix stack).  Each
// precision's variants live in their own translation unit (track_d.cu, track_dd.cu, track_qd.cu)
// so they compile in parallel.
#pragma once

#include <cstddef>
#include <cstdint>

namespace pp {
namespace dev {

constexpr int kHistDepth = 5;  // predictor history depth (reference tracker.cpp:87)
// slot-state field counts (enums F_*, R_*, D_* in track_impl.cuh)
constexpr int kIntFields = 14, kRealFields = 4, kDblFields = 3;

// StepEvent (tracker.hpp:62-69) as written by the device; layout-identical to pp_step_event
struct StepEventRec {
  unsigned long long path_id;
  double t;
  double h;
  uint32_t newton_iters;
  int8_t status;
  uint8_t accepted;
  uint8_t pad[2];
};
static_assert(sizeof(StepEventRec) == 32, "event record layout");

// Plan tables, device pointers (layouts documented in host.hpp, struct Plan)
struct PlanArgs {
  const int32_t* term_info;  // 4 per term
  const uint32_t* pos;
  const uint32_t* base;
  const double* coeff;       // per term: c_start (2L) then c_target (2L)
  // warp-cooperative evaluation (host.hpp Plan::term_slot / acc_off / acc_idx)
  const uint32_t* term_slot;
  const uint32_t* acc_off;
  const uint32_t* acc_idx;
  int n;                     // variables
  int n_polys;
  int n_terms;
  int n_slots;               // contribution slots of one evaluation
  // staging of the tables in shared memory (ctrl_eval_trip<..., kStage>): bytes of term_info,
  // pos, base, coeff, each a multiple of 16, and their total; the tables start at stage_offset
  // bytes into the dynamic shared memory
  uint32_t stage_bytes[5];
  uint32_t stage_offset;
};

// One persistent launch of the path tracker.
struct TrackArgs {
  PlanArgs plan;
  // start data: total degree (roots) or explicit list
  int total_degree;
  const uint32_t* degrees;
  const uint32_t* root_off;
  const double* roots;
  const double* explicit_x;
  // TrackConfig (tracker.hpp:29-46) + rank tolerance (linalg.hpp:44-52)
  double rtol, utol, h_init, h_min, h_max, expand, contract, div_bound, rank_tol;
  int max_newton, expand_after;
  uint32_t max_steps;
  // start-index range and refill counter.  The slot that draws refill number k (k < count) tracks
  // start index lo + ((k / shard_block) * shard_n + shard_r) * shard_block + k % shard_block: the
  // identity when shard_n == 1, else shard shard_r of a block-cyclic partition of [lo, hi)
  // among shard_n shards (multi-GPU load balance); its record is record k.
  unsigned long long lo, hi, count;
  unsigned long long shard_block, shard_n, shard_r;
  unsigned long long* next;
  unsigned long long* work;  // [0] evaluations, [1] least-squares solves issued
  // per-slot storage (S slots).  Planar arrays: element e, limb-plane p, slot s at ((e*P)+p)*S+s.
  uint32_t tmem_cols;  // tensor-memory columns per CTA of ctrl_eval_trip<..., kTmem = true>
  int lsq_spt;         // slots per thread of the q-cache solver (its grid covers n_active / lsq_spt)
  size_t S;         // slot stride of the planar arrays
  size_t n_active;  // slots [0, n_active) are launched (shrinks when the tail is compacted)
  int32_t* si;                  // integer state, field f at f*S + s (track_impl.cuh F_*)
  unsigned long long* spath;    // start index owned by the slot
  double* sr;                   // level-R scalars (t, h, t_next, final residual), planar real
  double* sd;                   // double scalars (residual, |dx|, |x|) at f*S + s
  double *x, *J, *Rm, *B, *Y, *xacc, *hx, *ht;
  // records, indexed by start index - lo
  double* rec_x;       // [rec][n][2L]
  double* rec_res;     // [rec][L]
  int8_t* rec_status;
  uint8_t* rec_reason;
  uint32_t *rec_steps, *rec_newton, *rec_rej;
  double* rec_div;     // [rec][4]: first, last, u_first, u_last of the terminal-divergence test
  uint8_t* rec_divflag;
  // step events (ProgressSink, tracker.hpp:62-70): one per step-control decision, appended at an
  // atomic cursor; ev == nullptr disables them.  Drained by the host after every graph launch.
  StepEventRec* ev;
  unsigned long long* ev_count;
  unsigned long long ev_cap;
};

// eval_system_batch for independent points (one thread per point)
struct EvalArgs {
  PlanArgs plan;
  uint32_t batch;
  const double* x;  // planar, S = batch: element v (n of them)
  const double* t;  // planar real, element 0
  double* sys;      // planar, element p (n_polys)
  double* jac;      // planar, element v*n_polys + p (column-major Jacobian)
};

// least_squares_solve for independent systems (one thread per system)
struct LsqArgs {
  int n;
  int m;       // rows (m >= n)
  uint32_t batch;
  double rank_tol;
  double* a;   // planar, element col*m + row (overwritten by Q)
  double* r;   // planar, packed upper triangle, n(n+1)/2
  double* b;   // planar, element row (m)
  double* y;   // planar scratch, n
  double* x;   // planar out, n
  uint8_t* ok;
};

constexpr int kCoopGroups[3] = {32, 8, 4};

// the corrector alone for independent (t, x) pairs (one thread per pair)
struct NewtonArgs {
  PlanArgs plan;
  uint32_t batch;
  int max_newton;
  double rtol, utol, rank_tol;
  double* x;        // planar, S = batch: element v (in: prediction, out: last iterate)
  const double* t;  // planar real, element 0
  double *J, *Rm, *B, *Y;  // planar scratch
  uint32_t* iters;
  uint8_t* corrected;
  uint8_t* singular;
};

struct Variant {
  int kmax;
  const void* ctrl_eval_trip;  // __global__ void(TrackArgs, unsigned* busy): control + evaluation
  const void* lsq_trip;   // __global__ void(TrackArgs)
  const void* step_trip;  // __global__ void(TrackArgs, unsigned* busy)
  const void* eval;       // __global__ void(EvalArgs)
  const void* lsq;        // __global__ void(LsqArgs)
  // tail mode, G lanes per slot for G = kCoopGroups[i] (32: a warp per slot)
  const void* eval_coop[3];   // __global__ void(TrackArgs)
  const void* lsq_coop[3];    // __global__ void(TrackArgs), Q and R in shared memory
  const void* lsq_coop_g[3];  // the same with Q and R in the global (tiled) arrays, for large n
  const void* ctrl_eval_tmem;  // ctrl_eval_trip with the open Jacobian row in tensor memory
  const void* lsq_tmem;        // lsq_trip with the Gram-Schmidt column in tensor memory
  const void* lsq_qcache;      // lsq_trip with q_i cached in tensor memory between dot and axpy
  const void* lsq_qcache_fuse; // the same with each axpy fused into the next dot product's row loop
  const void* newton;          // __global__ void(NewtonArgs): the corrector alone (set_prediction tests)
  const void* ctrl_eval_tmem_staged;  // ctrl_eval_tmem with the plan tables staged in shared memory by TMA
  const void* lsq_qcache_fuse_l2;     // lsq_qcache_fuse with L2 evict_last / evict_first policies on Q
};

// tail compaction: move the busy slots of [keep, n_active) into idle slots of [0, keep)
struct SlotArray {
  void* base;   // planar, plane p of slot s at base + (p*S + s) * bytes
  int planes;
  int bytes;    // 4 or 8
};
constexpr int kMaxSlotArrays = 12;
struct MoveArgs {
  SlotArray arr[kMaxSlotArrays];
  int n_arr;
  size_t S, n_active, keep;
  const int32_t* mode;  // plane F_MODE of the integer state
  unsigned* holes;      // idle slots below keep
  unsigned* movers;     // busy slots at or above keep
  unsigned* counts;     // [0] holes, [1] movers
};
void launch_compaction(const MoveArgs& m, void* stream);

// register-resident least-squares solvers, compiled for a few dimensions N (track_impl.cuh
// lsq_trip_reg): `stream` re-reads q_i for its axpy, `hold` keeps it in registers
struct LsqReg {
  int n;
  const void* stream;  // __global__ void(TrackArgs)
  const void* hold;    // __global__ void(TrackArgs)
};
const LsqReg* lsq_reg_d(int* count);
const LsqReg* lsq_reg_dd(int* count);

const Variant* variants_d(int* count);
const Variant* variants_dd(int* count);
const Variant* variants_qd(int* count);

}  // namespace dev
}  // namespace pp
