// device.cu -- host side of the CUDA path: plan upload, slot workspace, kernel selection and
// launch, record download.  No computation of the path happens here.

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>
#include <mutex>
#include <string>
#include <vector>

#include "device.hpp"
#include "kernels.hpp"

namespace pp {

namespace {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
T* dmalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  check(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
  return static_cast<T*>(p);
}

// a pair of timing events, destroyed on every path
struct EvPair {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  EvPair() {
    check(cudaEventCreate(&e0), "event");
    check(cudaEventCreate(&e1), "event");
  }
  EvPair(const EvPair&) = delete;
  EvPair& operator=(const EvPair&) = delete;
  ~EvPair() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  }
};

// device buffer owned for the duration of a kernel-level call (freed on every path)
template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t count) { p = dmalloc<T>(count); }
  explicit DevBuf(const std::vector<T>& v) {
    p = dmalloc<T>(v.size());
    if (!v.empty()) check(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// the allocation is padded to a multiple of 16 bytes (bulk copies move whole 16-byte units)
template <class T>
T* upload(const std::vector<T>& v) {
  const size_t bytes = (v.size() * sizeof(T) + 15) / 16 * 16;
  T* p = dmalloc<T>((bytes + sizeof(T) - 1) / sizeof(T));
  if (!v.empty()) check(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
  return p;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw CudaFailure("no CUDA device available (the tracker has no CPU fallback)");
    if (dev < 0 || dev >= count) throw CudaFailure("CUDA device index out of range");
    check(cudaGetDevice(&prev), "cudaGetDevice");
    check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// largest dimension the kernels take at level L: a 32-thread block of the evaluation kernel must
// hold its point and open Jacobian row (2n complex values per thread) in 200 KB of shared memory
uint32_t max_dim(int L) { return static_cast<uint32_t>((200 * 1024) / (32 * 2 * 2 * L * sizeof(double))); }

const dev::Variant* pick_variant(int prec, uint32_t n, uint32_t max_k) {
  int count = 0;
  const dev::Variant* v = prec == 0 ? dev::variants_d(&count)
                          : prec == 1 ? dev::variants_dd(&count)
                                      : dev::variants_qd(&count);
  const int L = prec == 0 ? 1 : (prec == 1 ? 2 : 4);
  if (n > max_dim(L)) return nullptr;
  const dev::Variant* best = nullptr;
  for (int i = 0; i < count; ++i) {
    if (v[i].kmax < static_cast<int>(std::max<uint32_t>(max_k, 2))) continue;
    if (best == nullptr || v[i].kmax < best->kmax) best = &v[i];
  }
  return best;
}

// Per (calling host thread, device) context, reused across calls: a grow-only workspace, the
// stream, timing events, a pinned mailbox and the pinned step-event staging buffer.  Concurrent
// track_all calls from different host threads (each on its own stream) never share one.
struct Ctx {
  int device = -1;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {};   // call phases: H2D, trips, D2H
  cudaEvent_t kev[4] = {};  // instrumented trips
  unsigned long long* mbox = nullptr;
  void* ev_host = nullptr;
  size_t ev_host_bytes = 0;

  explicit Ctx(int dev) : device(dev) {
    check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
    for (auto& e : ev) check(cudaEventCreate(&e), "event");
    for (auto& e : kev) check(cudaEventCreate(&e), "event");
    check(cudaMallocHost(&mbox, 4 * sizeof(unsigned long long)), "cudaMallocHost");
  }
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
  ~Ctx() {
    // best effort (the runtime may already be shutting down at thread / process exit)
    int prev = -1;
    if (cudaGetDevice(&prev) != cudaSuccess) return;
    cudaSetDevice(device);
    if (ws) cudaFree(ws);
    if (ev_host) cudaFreeHost(ev_host);
    if (mbox) cudaFreeHost(mbox);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : kev)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
    cudaSetDevice(prev);
  }
  void* workspace(size_t bytes) {
    if (ws_bytes < bytes) {
      check(cudaStreamSynchronize(stream), "workspace");
      if (ws) cudaFree(ws);
      ws = nullptr;
      ws_bytes = 0;
      check(cudaMalloc(&ws, bytes), "cudaMalloc(workspace)");
      ws_bytes = bytes;
    }
    return ws;
  }
  void* event_staging(size_t bytes) {
    if (ev_host_bytes < bytes) {
      if (ev_host) cudaFreeHost(ev_host);
      ev_host = nullptr;
      ev_host_bytes = 0;
      check(cudaMallocHost(&ev_host, bytes), "cudaMallocHost(events)");
      ev_host_bytes = bytes;
    }
    return ev_host;
  }
};
thread_local std::map<int, std::unique_ptr<Ctx>> t_ctx;

Ctx& context(int device) {
  auto& p = t_ctx[device];
  if (!p) p = std::make_unique<Ctx>(device);
  return *p;
}

// device properties, queried once per device
const cudaDeviceProp& device_props(int device) {
  static std::mutex mu;
  static std::map<int, cudaDeviceProp> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(device);
  if (it == cache.end()) {
    cudaDeviceProp p;
    check(cudaGetDeviceProperties(&p, device), "cudaGetDeviceProperties");
    it = cache.emplace(device, p).first;
  }
  return it->second;
}

// The dynamic shared memory limit of a kernel is raised, never lowered, under a lock: concurrent
// calls for systems of different sizes share kernels, and lowering the limit between another
// thread's check and its launch (or graph capture) would fail that launch.
void ensure_smem(const void* fn, size_t bytes, int device) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> cur;
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[{device, fn}];
  if (bytes <= c) return;
  check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)),
        "cudaFuncSetAttribute");
  c = bytes;
}

int occupancy(const void* fn, int block, size_t smem, int device) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, size_t>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(device, fn, block, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, smem), "occupancy");
  cache[key] = per_sm;
  return per_sm;
}

// scope guards of one tracking call
struct AsyncTemps {  // stream-ordered temporary allocations
  cudaStream_t stream;
  std::vector<void*> ptrs;
  void* alloc(size_t b) {
    void* p = nullptr;
    check(cudaMallocAsync(&p, b, stream), "cudaMallocAsync");
    ptrs.push_back(p);
    return p;
  }
  void release() {
    for (void* p : ptrs) cudaFreeAsync(p, stream);
    ptrs.clear();
  }
  ~AsyncTemps() { release(); }
};
struct GraphHolder {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
  }
  ~GraphHolder() { reset(); }
};
struct CaptureGuard {  // ends a capture an exception interrupted, so the stream stays usable
  cudaStream_t stream;
  bool active = false;
  ~CaptureGuard() {
    if (!active) return;
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(stream, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
  }
};

size_t align_up(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// carve consecutive aligned regions out of one allocation
struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    T* p = reinterpret_cast<T*>(base + off);
    off += align_up(count * sizeof(T));
    return p;
  }
};

dev::PlanArgs plan_args(const Plan& plan, const DevicePlan* dp);

}  // namespace

struct DevicePlan {
  int device = 0;
  int32_t* term_info = nullptr;
  uint32_t* pos = nullptr;
  uint32_t* base = nullptr;
  double* coeff = nullptr;
  uint32_t* term_slot = nullptr;
  uint32_t* acc_off = nullptr;
  uint32_t* acc_idx = nullptr;
};

namespace {
dev::PlanArgs plan_args(const Plan& plan, const DevicePlan* dp) {
  dev::PlanArgs pa{};
  pa.term_info = dp->term_info;
  pa.pos = dp->pos;
  pa.base = dp->base;
  pa.coeff = dp->coeff;
  pa.term_slot = dp->term_slot;
  pa.acc_off = dp->acc_off;
  pa.acc_idx = dp->acc_idx;
  pa.n_slots = static_cast<int>(plan.n_slots());
  pa.n = static_cast<int>(plan.dim);
  pa.n_polys = static_cast<int>(plan.n_polys);
  pa.n_terms = static_cast<int>(plan.n_terms());
  return pa;
}
}  // namespace

int device_count() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

bool device_supports(uint32_t n, uint32_t max_k) { return pick_variant(1, n, max_k) != nullptr; }

uint64_t shard_size(uint64_t lo, uint64_t hi, const TrackShard& sh) {
  if (hi <= lo) return 0;
  const uint64_t total = hi - lo;
  if (sh.count <= 1) return total;
  const uint64_t span = sh.block * sh.count, full = total / span, rem = total % span;
  const uint64_t first = sh.index * sh.block;
  return full * sh.block + (rem > first ? std::min<uint64_t>(sh.block, rem - first) : 0);
}

// ---------------------------------------------------------------------------------------------
// FP64 pipe throughput microbenchmark: the roofline denominator for the FP64-bound kernels.
// Eight independent DFMA chains per thread, one resident wave of blocks per SM.
// ---------------------------------------------------------------------------------------------
namespace {
__global__ void fp64_peak_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-3, a2 = a0 + 2e-3, a3 = a0 + 3e-3;
  double a4 = a0 + 4e-3, a5 = a0 + 5e-3, a6 = a0 + 6e-3, a7 = a0 + 7e-3;
  const double b = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
    a0 = __fma_rn(a0, b, c);
    a1 = __fma_rn(a1, b, c);
    a2 = __fma_rn(a2, b, c);
    a3 = __fma_rn(a3, b, c);
    a4 = __fma_rn(a4, b, c);
    a5 = __fma_rn(a5, b, c);
    a6 = __fma_rn(a6, b, c);
    a7 = __fma_rn(a7, b, c);
  }
  const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains alive
}
}  // namespace

// ---------------------------------------------------------------------------------------------
// tail compaction (the paper's active-path compaction): once the start counter
// is exhausted, busy slots above `keep` move into idle slots below it, so the remaining trips
// launch ceil(keep / block) blocks of densely packed warps.  Slot order does not matter: every
// per-path result is independent of which slot runs it.
// ---------------------------------------------------------------------------------------------
namespace dev {
namespace {
__global__ void classify_slots(const MoveArgs m) {
  const size_t s = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= m.n_active) return;
  const bool busy = m.mode[s] != 4;  // M_DONE
  if (s < m.keep && !busy) m.holes[atomicAdd(m.counts, 1u)] = static_cast<unsigned>(s);
  if (s >= m.keep && busy) m.movers[atomicAdd(m.counts + 1, 1u)] = static_cast<unsigned>(s);
}
__global__ void move_slots(const MoveArgs m) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m.counts[1]) return;
  const size_t from = m.movers[i], to = m.holes[i];
  for (int k = 0; k < m.n_arr; ++k) {
    const SlotArray& a = m.arr[k];
    for (int p = 0; p < a.planes; ++p) {
      const size_t o = static_cast<size_t>(p) * m.S;
      if (a.bytes == 8) {
        double* b = static_cast<double*>(a.base);
        b[o + to] = b[o + from];
      } else {
        int32_t* b = static_cast<int32_t*>(a.base);
        b[o + to] = b[o + from];
      }
    }
  }
}
}  // namespace

void launch_compaction(const MoveArgs& m, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  check(cudaMemsetAsync(m.counts, 0, 2 * sizeof(unsigned), st), "memset counts");
  const unsigned b = 256;
  classify_slots<<<static_cast<unsigned>((m.n_active + b - 1) / b), b, 0, st>>>(m);
  move_slots<<<static_cast<unsigned>((m.n_active - m.keep + b - 1) / b + 1), b, 0, st>>>(m);
  check(cudaGetLastError(), "compaction");
}
}  // namespace dev

// Create the device context and this thread's stream / workspace context, and load the tracking
// kernels (module loading is lazy otherwise: the first launch of each kernel would pay for it).
void device_init(int device) {
  DeviceGuard g(device);
  check(cudaFree(nullptr), "context");
  (void)device_props(device);
  (void)context(device);
  for (auto fn : {&dev::variants_d, &dev::variants_dd, &dev::variants_qd}) {
    int cnt = 0;
    const dev::Variant* v = fn(&cnt);
    for (int i = 0; i < cnt; ++i)
      for (const void* k : {v[i].ctrl_eval_trip, v[i].lsq_trip, v[i].step_trip, v[i].eval, v[i].lsq, v[i].eval_coop[0],
                            v[i].eval_coop[1], v[i].eval_coop[2], v[i].lsq_coop[0], v[i].lsq_coop[1], v[i].lsq_coop[2],
                            v[i].lsq_coop_g[0], v[i].lsq_coop_g[1], v[i].lsq_coop_g[2], v[i].ctrl_eval_tmem,
                            v[i].lsq_qcache, v[i].lsq_qcache_fuse, v[i].ctrl_eval_tmem_staged, v[i].lsq_qcache_fuse_l2}) {
        cudaFuncAttributes at;
        check(cudaFuncGetAttributes(&at, k), "kernel load");
      }
  }
  int cnt = 0;
  const dev::LsqReg* lr = dev::lsq_reg_d(&cnt);
  for (int i = 0; i < cnt; ++i) {
    cudaFuncAttributes at;
    check(cudaFuncGetAttributes(&at, lr[i].hold), "kernel load");
  }
  for (const void* k : {reinterpret_cast<const void*>(&dev::classify_slots), reinterpret_cast<const void*>(&dev::move_slots)}) {
    cudaFuncAttributes at;
    check(cudaFuncGetAttributes(&at, k), "kernel load");
  }
}

double device_fp64_peak(int device) {
  DeviceGuard g(device);
  cudaDeviceProp prop;
  check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  const int block = 256, per_sm = 8, iters = 1 << 14;
  const int blocks = prop.multiProcessorCount * per_sm;
  DevBuf<double> out(blocks);
  EvPair ev;
  fp64_peak_kernel<<<blocks, block>>>(out.p, iters);  // warm-up
  check(cudaEventRecord(ev.e0), "event");
  const int reps = 5;
  for (int r = 0; r < reps; ++r) fp64_peak_kernel<<<blocks, block>>>(out.p, iters);
  check(cudaEventRecord(ev.e1), "event");
  check(cudaEventSynchronize(ev.e1), "fp64 peak kernel");
  float ms = 0;
  check(cudaEventElapsedTime(&ms, ev.e0, ev.e1), "event time");
  const double ops = static_cast<double>(reps) * blocks * block * iters * 8.0;
  return ops / (ms / 1e3);
}

DevicePlan* device_plan_upload(const Plan& plan, int device) {
  DeviceGuard g(device);
  auto* dp = new DevicePlan;
  dp->device = device;
  try {
    dp->term_info = upload(plan.term_info);
    dp->pos = upload(plan.pos);
    dp->base = upload(plan.base);
    dp->coeff = upload(plan.coeff);
    dp->term_slot = upload(plan.term_slot);
    dp->acc_off = upload(plan.acc_off);
    dp->acc_idx = upload(plan.acc_idx);
  } catch (...) {
    device_plan_free(dp);
    throw;
  }
  return dp;
}

void device_plan_free(DevicePlan* dp) {
  if (dp == nullptr) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(dp->device);
  cudaFree(dp->term_info);
  cudaFree(dp->pos);
  cudaFree(dp->base);
  cudaFree(dp->coeff);
  cudaFree(dp->term_slot);
  cudaFree(dp->acc_off);
  cudaFree(dp->acc_idx);
  if (prev >= 0) cudaSetDevice(prev);
  delete dp;
}

// launch geometry of one tracking run: S slots in blocks of kBlock threads
constexpr int kBlock = 128;

size_t env_size(const char* name, size_t dflt) {
  const char* v = std::getenv(name);
  if (v == nullptr || *v == '\0') return dflt;
  return static_cast<size_t>(std::strtoull(v, nullptr, 10));
}

void device_track(const Plan& plan, DevicePlan* dp, const Starts& st, const pp_track_config& cfg,
                  uint64_t lo, uint64_t hi, const TrackShard& shard, const EventSink& sink, int device,
                  pp_records* out, pp_run_stats* stats) {
  auto wall0 = std::chrono::steady_clock::now();
  DeviceGuard g(device);
  const uint32_t n = plan.dim;
  const uint32_t L = plan.L;
  const dev::Variant* var = pick_variant(plan.prec, n, plan.max_k);
  if (var == nullptr) throw InvalidArgument("system dimension / monomial size beyond the compiled kernels (KMAX 16; n <= 97 in dd)");
  const uint64_t count = shard_size(lo, hi, shard);  // records of this call

  const cudaDeviceProp& prop = device_props(device);
  const size_t per_thread_smem = static_cast<size_t>(2) * n * 2 * L * sizeof(double);
  int tblock = static_cast<int>(std::min<size_t>(128, std::max<size_t>(32, env_size("PP200_TRIP_BLOCK", kBlock))));
  while (tblock > 32 && static_cast<size_t>(tblock) * per_thread_smem > 200 * 1024) tblock /= 2;
  // the evaluation kernel may run narrower blocks than the others (its shared memory -- point
  // and open Jacobian row per thread -- is what limits its occupancy)
  int eblock = static_cast<int>(std::min<size_t>(tblock, std::max<size_t>(32, env_size("PP200_EVAL_BLOCK", tblock))));
  while (tblock % eblock != 0) eblock /= 2;
  // the open Jacobian row in tensor memory (n*4L 32-bit columns per thread, at most 128; a CTA of
  // four warps covers the four TMEM lane quarters, four CTAs use all 512 columns); PP200_TMEM=0
  // keeps it in shared memory
  bool tmem = env_size("PP200_TMEM", 1) != 0 && static_cast<size_t>(n) * 4 * L <= 128 && eblock == 128;
  uint32_t tmem_cols = 32;
  while (tmem_cols < static_cast<uint32_t>(n) * 4 * L) tmem_cols *= 2;
  int eval_ctas = 0;  // resident CTAs per SM of the TMEM evaluation
  if (tmem) {
    // every resident CTA must get its columns at once (512 per SM), or tcgen05.alloc would stall
    ensure_smem(var->ctrl_eval_tmem, eblock * per_thread_smem / 2, device);
    eval_ctas = occupancy(var->ctrl_eval_tmem, eblock, eblock * per_thread_smem / 2, device);
    tmem = static_cast<uint32_t>(eval_ctas) * tmem_cols <= 512;
  }
  const void* ctrl_eval_fn = tmem ? var->ctrl_eval_tmem : var->ctrl_eval_trip;
  size_t eval_smem = static_cast<size_t>(eblock) * per_thread_smem / (tmem ? 2 : 1);
  // PP200_STAGE_TABLES (TMEM evaluation; default 1 in complex double, 0 otherwise): the plan tables
  // go to shared memory by bulk TMA copies when each CTA starts, and the evaluation reads them from
  // there.  Cyclic-10 d: 254 k -> 281 k paths/s.  Cyclic-10 dd: evaluation 6.14 -> 6.24 s per
  // 262,144 paths (the broadcast table reads hit L1 anyway, and the tables' shared memory shrinks
  // the L1 that holds the Speelpenning prefix stack), so double-double reads them from global memory.
  dev::PlanArgs staged_plan = plan_args(plan, dp);
  if (tmem && env_size("PP200_STAGE_TABLES", L == 1 ? 1 : 0) != 0) {
    auto r16 = [](size_t b) { return static_cast<uint32_t>((b + 15) / 16 * 16); };
    staged_plan.stage_bytes[0] = r16(plan.term_info.size() * sizeof(int32_t));
    staged_plan.stage_bytes[1] = r16(plan.pos.size() * sizeof(uint32_t));
    staged_plan.stage_bytes[2] = r16(plan.base.size() * sizeof(uint32_t));
    staged_plan.stage_bytes[3] = r16(plan.coeff.size() * sizeof(double));
    staged_plan.stage_bytes[4] =
        staged_plan.stage_bytes[0] + staged_plan.stage_bytes[1] + staged_plan.stage_bytes[2] + staged_plan.stage_bytes[3];
    staged_plan.stage_offset = static_cast<uint32_t>(eval_smem);
    // only while the tables do not cost a resident CTA (1 KB per CTA is reserved by the runtime)
    if ((eval_smem + staged_plan.stage_bytes[4] + 1024) * static_cast<size_t>(eval_ctas) <=
        prop.sharedMemPerMultiprocessor) {
      eval_smem += staged_plan.stage_bytes[4];
      ctrl_eval_fn = var->ctrl_eval_tmem_staged;
    }
  }
  // least squares: the column being orthogonalised in shared memory, or (PP200_LSQ_TMEM=1, n*4L <= 128)
  // in tensor memory with 256-thread CTAs, two per SM (256 TMEM columns each), leaving L1 to Q
  bool lsq_tm = env_size("PP200_LSQ_TMEM", 0) != 0 && static_cast<size_t>(n) * 4 * L <= 128 && tblock == 128;
  if (lsq_tm) lsq_tm = occupancy(var->lsq_tmem, 256, 0, device) <= 2;  // more CTAs than TMEM columns would stall
  const void* lsq_fn = lsq_tm ? var->lsq_tmem : var->lsq_trip;
  // register-resident solver for the compiled dimensions (PP200_LSQ_REG: 0 off, 1 stream, 2 hold q_i;
  // default 2 in complex double, where it halves the solver's HBM traffic: lsq 0.86 -> 0.53 s on
  // 262,144 cyclic-10 paths)
  const void* lsq_reg = nullptr;
  if (!lsq_tm && tblock == 128 && plan.prec <= 1) {
    const size_t mode = env_size("PP200_LSQ_REG", plan.prec == 0 ? 2 : 0);
    int cnt = 0;
    const dev::LsqReg* lr = plan.prec == 0 ? dev::lsq_reg_d(&cnt) : dev::lsq_reg_dd(&cnt);
    for (int i = 0; i < cnt && mode != 0; ++i)
      if (lr[i].n == static_cast<int>(n)) lsq_reg = mode == 1 ? lr[i].stream : lr[i].hold;
  }
  if (lsq_reg) lsq_fn = lsq_reg;
  // PP200_LSQ_QCACHE (default 1 for n*4L <= 128): the column in shared memory and q_i cached in
  // TMEM between its dot product and its axpy (128 columns per CTA; the shared memory request is
  // padded so that at most four CTAs are resident per SM and every tcgen05.alloc succeeds at once).
  // Measured on cyclic-10 dd: lsq 5.47 -> 5.33 s per 131,072 paths.
  // Double-double only: in complex double the cache costs more than the re-read it saves
  // (rand32 d: 3,610 -> 3,102 paths/s).
  const bool lsq_qc = !lsq_tm && !lsq_reg && tblock == 128 && env_size("PP200_LSQ_QCACHE", L == 2 ? 1 : 0) != 0 &&
                      static_cast<size_t>(n) * 4 * L <= 128;
  // PP200_LSQ_FUSE (default 1): with the q-cache, each axpy shares its row loop with the next dot
  // product (cyclic-10 dd: lsq 9.73 -> 9.54 s per 262,144 paths; cyclic-8 dd +2.3 %)
  if (lsq_qc) lsq_fn = env_size("PP200_LSQ_FUSE", 1) != 0 ? var->lsq_qcache_fuse : var->lsq_qcache;
  // PP200_LSQ_L2HINT (default 1): the fused solver with L2 eviction policies on Q, the first half of
  // the columns (the most re-read) evict_last, the rest evict_first: DRAM per launch 2.93 -> 2.46 GB
  // on a full-occupancy cyclic-10 dd trip (L2 hit rate 20 -> 29 %), run time unchanged
  if (lsq_qc && env_size("PP200_LSQ_FUSE", 1) != 0 && env_size("PP200_LSQ_L2HINT", 1) != 0) lsq_fn = var->lsq_qcache_fuse_l2;
  const int lblock = lsq_tm ? 256 : tblock;
  size_t lsq_smem = (lsq_tm || lsq_reg) ? 0 : static_cast<size_t>(tblock) * per_thread_smem / 2;
  if (lsq_qc) lsq_smem = std::max<size_t>(lsq_smem, (prop.sharedMemPerMultiprocessor / 5) + 1024);
  ensure_smem(ctrl_eval_fn, eval_smem, device);
  ensure_smem(lsq_fn, lsq_smem, device);
  // slots: PP200_SLOTS_PER_SM per SM (default 512; 1024 in complex double, whose kernels are
  // memory-latency bound and want more warps), never more than the paths (whole blocks)
  const size_t per_sm = std::max<size_t>(tblock, env_size("PP200_SLOTS_PER_SM", L == 1 ? 1024 : 512));
  uint64_t blocks = (per_sm / tblock) * static_cast<uint64_t>(prop.multiProcessorCount);
  blocks = std::min<uint64_t>(blocks, (count + tblock - 1) / tblock);
  blocks = std::max<uint64_t>(blocks, 1);
  const size_t S = blocks * tblock;

  const size_t cw = 2 * L;  // doubles per complex
  // planar slot arrays are addressed with 32-bit offsets (track_impl.cuh, Planar::at)
  if (static_cast<size_t>(dev::kHistDepth) * n * cw * S >= (static_cast<size_t>(1) << 32) ||
      static_cast<size_t>(n) * n * cw * S >= (static_cast<size_t>(1) << 32))
    throw InvalidArgument("track_all: slot arrays exceed 2^32 doubles (lower PP200_SLOTS_PER_SM)");
  const size_t nJ = static_cast<size_t>(n) * n, nR = static_cast<size_t>(n) * (n + 1) / 2;
  const size_t kH = dev::kHistDepth;
  const size_t graph_trips = std::max<size_t>(1, env_size("PP200_GRAPH_TRIPS", 16));
  // step events: at most one per busy slot and trip, so graph_trips * S per drain
  const uint64_t ev_cap = sink.fn ? static_cast<uint64_t>(graph_trips) * S : 0;
  size_t bytes = 0;
  auto room = [&](size_t b) { bytes += align_up(b); };
  room(dev::kIntFields * S * 4);
  room(S * 8);
  room(dev::kRealFields * L * S * 8);
  room(dev::kDblFields * S * 8);
  for (size_t elems : {static_cast<size_t>(n), nJ, nR, static_cast<size_t>(n), static_cast<size_t>(n),
                       static_cast<size_t>(n), kH * n})
    room(elems * cw * S * 8);
  room(kH * L * S * 8);
  const size_t rec_bytes_x = count * n * cw * sizeof(double);
  room(rec_bytes_x);
  room(count * L * 8);
  room(count);
  room(count);
  room(count * 4);
  room(count * 4);
  room(count * 4);
  room(count * 4 * 8);
  room(count);
  room(64);
  room(graph_trips * 4);
  room(ev_cap * sizeof(dev::StepEventRec));
  room((2 * S + 2) * sizeof(unsigned));  // compaction lists
  Ctx& cx = context(device);
  Carver cv{static_cast<char*>(cx.workspace(bytes))};

  dev::TrackArgs a{};
  a.plan = staged_plan;
  a.total_degree = st.total_degree ? 1 : 0;
  a.rtol = cfg.residual_tol;
  a.utol = cfg.update_tol;
  a.h_init = cfg.h_init;
  a.h_min = cfg.h_min;
  a.h_max = cfg.h_max;
  a.expand = cfg.expand;
  a.contract = cfg.contract;
  a.div_bound = cfg.divergence_bound;
  a.rank_tol = default_rank_tol(plan.prec);
  a.max_newton = cfg.max_newton;
  a.expand_after = cfg.expand_after;
  a.max_steps = cfg.max_steps;
  a.lo = lo;
  a.hi = hi;
  a.count = count;
  a.shard_block = shard.count > 1 ? shard.block : 1;
  a.shard_n = shard.count > 1 ? shard.count : 1;
  a.shard_r = shard.count > 1 ? shard.index : 0;
  a.S = S;
  a.si = cv.take<int32_t>(dev::kIntFields * S);
  a.spath = cv.take<unsigned long long>(S);
  a.sr = cv.take<double>(dev::kRealFields * L * S);
  a.sd = cv.take<double>(dev::kDblFields * S);
  a.x = cv.take<double>(n * cw * S);
  a.J = cv.take<double>(nJ * cw * S);
  a.Rm = cv.take<double>(nR * cw * S);
  a.B = cv.take<double>(n * cw * S);
  a.Y = cv.take<double>(n * cw * S);
  a.xacc = cv.take<double>(n * cw * S);
  a.hx = cv.take<double>(kH * n * cw * S);
  a.ht = cv.take<double>(kH * L * S);
  a.rec_x = cv.take<double>(count * n * cw);
  a.rec_res = cv.take<double>(count * L);
  a.rec_status = cv.take<int8_t>(count);
  a.rec_reason = cv.take<uint8_t>(count);
  a.rec_steps = cv.take<uint32_t>(count);
  a.rec_newton = cv.take<uint32_t>(count);
  a.rec_rej = cv.take<uint32_t>(count);
  a.rec_div = cv.take<double>(count * 4);
  a.rec_divflag = cv.take<uint8_t>(count);
  a.next = cv.take<unsigned long long>(8);
  a.work = a.next + 2;
  a.ev_count = a.next + 4;
  unsigned* busy = cv.take<unsigned>(graph_trips);
  a.ev = ev_cap ? cv.take<dev::StepEventRec>(ev_cap) : nullptr;
  a.ev_cap = ev_cap;
  unsigned* holes = cv.take<unsigned>(2 * S + 2);
  dev::StepEventRec* ev_host = ev_cap ? static_cast<dev::StepEventRec*>(cx.event_staging(ev_cap * sizeof(dev::StepEventRec)))
                                      : nullptr;

  cudaStream_t stream = cx.stream;
  cudaEvent_t* e = cx.ev;  // e[0] H2D e[1] trips e[2] D2H e[3]
  unsigned long long* mbox = cx.mbox;  // pinned: [0] busy slots, [1] start counter, [2] events
  AsyncTemps temps{stream};
  GraphHolder gh;
  CaptureGuard capg{stream};

  // start tables (small): uploaded per call; explicit start lists only for [lo, hi)
  uint64_t h2d = 0;
  auto up = [&](const void* src, size_t b) -> void* {
    void* p = temps.alloc(b == 0 ? 1 : b);
    if (b) check(cudaMemcpyAsync(p, src, b, cudaMemcpyHostToDevice, stream), "H2D");
    h2d += b;
    return p;
  };
  check(cudaEventRecord(e[0], stream), "event");
  if (st.total_degree) {
    a.degrees = static_cast<const uint32_t*>(up(st.degrees.data(), st.degrees.size() * 4));
    a.root_off = static_cast<const uint32_t*>(up(st.root_off.data(), st.root_off.size() * 4));
    a.roots = static_cast<const double*>(up(st.roots.data(), st.roots.size() * 8));
  } else {
    a.explicit_x = static_cast<const double*>(up(st.explicit_x.data() + lo * n * cw, (hi - lo) * n * cw * 8));
  }
  check(cudaEventRecord(e[1], stream), "event");
  check(cudaMemsetAsync(a.si, 0, dev::kIntFields * S * 4, stream), "memset");  // all slots M_IDLE
  check(cudaMemsetAsync(a.next, 0, 8 * sizeof(unsigned long long), stream), "memset");

  // hand the step events produced so far to the sink and reset the ring (stream is idle here)
  uint64_t n_events = 0;
  auto drain_events = [&]() {
    if (!ev_cap) return;
    check(cudaMemcpyAsync(mbox + 2, a.ev_count, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream), "D2H");
    check(cudaStreamSynchronize(stream), "events");
    const uint64_t ne = mbox[2];
    if (ne > ev_cap) throw CudaFailure("step-event ring overflow");
    if (ne == 0) return;
    check(cudaMemcpyAsync(ev_host, a.ev, ne * sizeof(dev::StepEventRec), cudaMemcpyDeviceToHost, stream), "D2H");
    check(cudaMemsetAsync(a.ev_count, 0, sizeof(unsigned long long), stream), "memset");
    check(cudaStreamSynchronize(stream), "events");
    sink.fn(reinterpret_cast<const pp_step_event*>(ev_host), ne, sink.user);
    n_events += ne;
  };

  uint64_t trips = 0, launches = 0, compactions = 0, per_graph_launches = 0;
  float kms[3] = {0, 0, 0};  // eval (thread mode: control + evaluation), lsq, tail-mode control
  a.n_active = S;
  a.tmem_cols = tmem_cols;
  // PP200_LSQ_SPT: slots per thread of the q-cache solver (1 or 2)
  a.lsq_spt = lsq_qc ? static_cast<int>(std::min<size_t>(2, std::max<size_t>(1, env_size("PP200_LSQ_SPT", 1)))) : 1;
  {
    const dim3 blk(tblock);
    dim3 grid(static_cast<unsigned>(blocks));
    auto egrid = [&]() { return dim3(grid.x * static_cast<unsigned>(tblock / eblock)); };
    void* targs[] = {&a};

    // tail mode (PP200_TAIL_SLOTS, default 32 per SM; 0 disables): once compaction has shrunk the
    // launch to at most that many slots, each remaining path gets a whole warp (eval_coop /
    // lsq_coop), bitwise identical to the thread-per-path kernels
    const size_t el = static_cast<size_t>(2) * L * sizeof(double);  // bytes per complex value
    const size_t ecoop_slot = (static_cast<size_t>(n) + plan.n_slots()) * el;
    // Q and R in shared memory while they take at most PP200_COOP_SMEM_KB (4) KB per slot, else
    // left in the global arrays (more slots per SM)
    const bool coop_global = static_cast<size_t>(n) * n * el > env_size("PP200_COOP_SMEM_KB", 4) * 1024;
    const size_t lcoop_slot =
        (coop_global ? static_cast<size_t>(4) * n : static_cast<size_t>(n) * n + 4 * n + n * (n + 1) / 2) * el;
    // lanes per slot (G = 32, 8 or 4; G < 32 packs 32 / G slots into a warp), chosen per kernel.  A
    // warp per slot gives each path the lowest trip latency, which is what the last few paths of a
    // run need; with many slots per SM, smaller groups keep more lanes of the solver busy (the
    // reference's sequential sums run on two lanes of the group, its row operations on all of
    // them).  The evaluation keeps a warp per slot: its per-slot contribution buffer is large, so
    // packing slots would cut the warps per SM instead.  PP200_COOP_GROUP fixes the solver's G,
    // PP200_COOP_GROUP_EVAL the evaluation's; by default the solver uses G = 8 from
    // PP200_COOP_G8_PER_SM (8) busy slots per SM up.
    // warps per block of a tail-mode kernel with per-slot shared memory per_slot and group index
    // gi (at most 4, within 200 KB; 0 if one warp does not fit)
    auto coop_wpb = [&](size_t per_slot, int gi) {
      const size_t per_warp = per_slot * static_cast<size_t>(32 / dev::kCoopGroups[gi]);
      return static_cast<int>(std::min<size_t>(4, (200 * 1024) / per_warp));
    };
    auto group_index = [](size_t g) { return g == 8 ? 1 : g == 4 ? 2 : 0; };
    const size_t g8_per_sm = env_size("PP200_COOP_G8_PER_SM", 8);
    const int lsq_gi_env = group_index(env_size("PP200_COOP_GROUP", 0)), eval_gi_env = group_index(env_size("PP200_COOP_GROUP_EVAL", 32));
    const bool lsq_g_fixed = env_size("PP200_COOP_GROUP", 0) != 0;
    auto lsq_gi = [&](size_t active) -> int {
      int gi = lsq_g_fixed ? lsq_gi_env : (active >= g8_per_sm * static_cast<size_t>(prop.multiProcessorCount) ? 1 : 0);
      while (gi > 0 && coop_wpb(lcoop_slot, gi) < 1) --gi;
      return gi;
    };
    auto eval_gi = [&](size_t) -> int {
      int gi = eval_gi_env;
      while (gi > 0 && coop_wpb(ecoop_slot, gi) < 1) --gi;
      return gi;
    };
    // tail mode needs a warp per slot to fit (G = 32)
    const bool coop_ok = coop_wpb(ecoop_slot, 0) >= 1 && coop_wpb(lcoop_slot, 0) >= 1;
    for (int gi = 0; gi < 3 && coop_ok; ++gi) {
      const size_t spw = static_cast<size_t>(32 / dev::kCoopGroups[gi]);
      const int ew = coop_wpb(ecoop_slot, gi), lw = coop_wpb(lcoop_slot, gi);
      if (ew >= 1) ensure_smem(var->eval_coop[gi], ew * spw * ecoop_slot, device);
      if (lw >= 1) ensure_smem(coop_global ? var->lsq_coop_g[gi] : var->lsq_coop[gi], lw * spw * lcoop_slot, device);
    }
    const size_t tail_slots = env_size("PP200_TAIL_SLOTS", 32 * static_cast<size_t>(prop.multiProcessorCount));
    // PP200_FORCE_COOP=1 runs every trip in tail mode (used by the parity tests)
    // small runs (no more paths than tail slots) start in tail mode: a warp per path spreads a
    // few thousand paths over every SM instead of packing them into a few blocks
    // Whole quad-double runs stay in tail mode: a thread per path leaves a few warps per SM for
    // its per-thread working set (katsura-12 qd: 80.5 s thread per path against 21.6 s with
    // groups of 8 lanes).  Large double-double systems do not: rand32 dd over all 65,536 paths
    // runs at 408 paths/s a thread per path against 290 in tail mode (a 8,192-path sample
    // favoured tail mode, 184 vs 148: its tail dominates).
    const bool coop_whole_run = env_size("PP200_COOP_WHOLE_RUN", 1) != 0 && plan.prec == 2;
    bool coop = (env_size("PP200_FORCE_COOP", 0) != 0 || coop_whole_run || (tail_slots > 0 && count <= tail_slots)) &&
                coop_ok;
    // one trip = control (step control, prediction, finalize, refill) followed by the heavy
    // operation of every busy slot.  Thread-per-path mode fuses the control into the evaluation
    // kernel (ctrl_eval_trip) and runs lsq_trip; tail mode runs step_trip, eval_coop, lsq_coop.
    // The control part counts the slots with work in this trip into *busy_ptr.  With events
    // (instrumented mode) the three phases are bracketed: ev[0] ctrl ev[1] eval ev[2] lsq ev[3].
    auto launch_trip = [&](unsigned* busy_ptr, cudaEvent_t* ev) {
      void* args[] = {&a, &busy_ptr};
      if (ev) check(cudaEventRecord(ev[0], stream), "event");
      if (coop) {
        check(cudaLaunchKernel(var->step_trip, grid, blk, args, 0, stream), "launch step_trip");
        if (ev) check(cudaEventRecord(ev[1], stream), "event");
        const int egi = eval_gi(a.n_active), lgi = lsq_gi(a.n_active);
        const size_t espw = static_cast<size_t>(32 / dev::kCoopGroups[egi]);
        const size_t lspw = static_cast<size_t>(32 / dev::kCoopGroups[lgi]);
        const int ew = coop_wpb(ecoop_slot, egi), lw = coop_wpb(lcoop_slot, lgi);
        const unsigned eb = static_cast<unsigned>((a.n_active + ew * espw - 1) / (ew * espw));
        const unsigned lb = static_cast<unsigned>((a.n_active + lw * lspw - 1) / (lw * lspw));
        check(cudaLaunchKernel(var->eval_coop[egi], dim3(eb), dim3(32 * ew), targs, ew * espw * ecoop_slot, stream),
              "launch eval_coop");
        if (ev) check(cudaEventRecord(ev[2], stream), "event");
        check(cudaLaunchKernel(coop_global ? var->lsq_coop_g[lgi] : var->lsq_coop[lgi], dim3(lb), dim3(32 * lw), targs,
                               lw * lspw * lcoop_slot, stream),
              "launch lsq_coop");
      } else {
        if (ev) check(cudaEventRecord(ev[1], stream), "event");
        check(cudaLaunchKernel(ctrl_eval_fn, egrid(), dim3(eblock), args, eval_smem, stream),
              "launch ctrl_eval_trip");
        if (ev) check(cudaEventRecord(ev[2], stream), "event");
        const size_t per_block = static_cast<size_t>(lblock) * a.lsq_spt;
        check(cudaLaunchKernel(lsq_fn, dim3(static_cast<unsigned>((a.n_active + per_block - 1) / per_block)), dim3(lblock),
                               targs, lsq_smem, stream),
              "launch lsq_trip");
      }
      if (ev) check(cudaEventRecord(ev[3], stream), "event");
      launches += coop ? 3 : 2;
    };

    // tail compaction once the start counter is exhausted and at most compact_frac of the
    // launched slots are busy (PP200_COMPACT=0 disables it)
    const bool compact = env_size("PP200_COMPACT", 1) != 0;
    // compact when at most this fraction of the launched slots is busy (PP200_COMPACT_PCT)
    const double compact_frac = static_cast<double>(std::min<size_t>(99, env_size("PP200_COMPACT_PCT", 95))) / 100.0;
    auto maybe_compact = [&](unsigned long long nbusy, unsigned long long started) -> bool {
      if (!compact || started < count || nbusy == 0 ||
          static_cast<double>(nbusy) > compact_frac * static_cast<double>(a.n_active))
        return false;
      const size_t keep = (nbusy + tblock - 1) / tblock * tblock;
      if (keep >= a.n_active) return false;
      dev::MoveArgs m{};
      const size_t nL = n * cw;
      const dev::SlotArray arrs[] = {
          {a.si, dev::kIntFields, 4}, {a.spath, 1, 8}, {a.sr, dev::kRealFields * static_cast<int>(L), 8},
          {a.sd, dev::kDblFields, 8}, {a.x, static_cast<int>(nL), 8}, {a.xacc, static_cast<int>(nL), 8},
          {a.hx, static_cast<int>(kH * nL), 8}, {a.ht, static_cast<int>(kH * L), 8}};
      m.n_arr = static_cast<int>(sizeof(arrs) / sizeof(arrs[0]));
      for (int i = 0; i < m.n_arr; ++i) m.arr[i] = arrs[i];
      m.S = S;
      m.n_active = a.n_active;
      m.keep = keep;
      m.mode = a.si;  // plane F_MODE = 0
      m.holes = holes;
      m.movers = holes + S;
      m.counts = holes + 2 * S;
      dev::launch_compaction(m, stream);
      a.n_active = keep;
      grid = dim3(static_cast<unsigned>(keep / tblock));
      coop = coop || (tail_slots > 0 && coop_ok && keep <= tail_slots);
      ++compactions;
      launches += 2;
      return true;
    };

    if (env_size("PP200_KERNEL_TIMING", 0) != 0) {
      // instrumented mode: plain launches bracketed by events, per-kernel device time accumulated
      cudaEvent_t* ev = cx.kev;
      // PP200_TRIP_LOG=<file>: one line per trip (trip, busy slots, eval/lsq/control ms, launched
      // slots, tail mode)
      const char* log_path = std::getenv("PP200_TRIP_LOG");
      std::unique_ptr<FILE, int (*)(FILE*)> trip_log((log_path && *log_path) ? std::fopen(log_path, "a") : nullptr,
                                                     [](FILE* f) { return f ? std::fclose(f) : 0; });
      for (;;) {
        check(cudaMemsetAsync(busy, 0, sizeof(unsigned), stream), "memset busy");
        const size_t trip_active = a.n_active;
        const bool trip_coop = coop;
        launch_trip(busy, ev);
        check(cudaMemcpyAsync(mbox, busy, sizeof(unsigned), cudaMemcpyDeviceToHost, stream), "D2H");
        check(cudaMemcpyAsync(mbox + 1, a.next, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream), "D2H");
        check(cudaStreamSynchronize(stream), "tracker trip");
        const unsigned long long nbusy = *reinterpret_cast<unsigned*>(mbox);
        float tms[3] = {0, 0, 0};  // ctrl, eval (thread mode: control + evaluation), lsq
        for (int k = 0; k < 3; ++k) check(cudaEventElapsedTime(&tms[k], ev[k], ev[k + 1]), "event time");
        kms[0] += tms[1];
        kms[1] += tms[2];
        kms[2] += tms[0];
        if (trip_log)
          std::fprintf(trip_log.get(), "%llu %llu %.4f %.4f %.4f %llu %d\n", static_cast<unsigned long long>(trips), nbusy,
                       tms[1], tms[2], tms[0], static_cast<unsigned long long>(trip_active), trip_coop ? 1 : 0);
        ++trips;
        drain_events();
        if (nbusy == 0) break;
        maybe_compact(nbusy, mbox[1]);
      }
    } else {
      // one trip = evaluate, solve, control; trips are captured G at a time into a CUDA graph
      // whose last control kernel reports how many slots are still busy.  The graph is
      // re-captured when compaction shrinks the launch.
      auto capture = [&]() {
        gh.reset();
        check(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "capture");
        capg.active = true;
        check(cudaMemsetAsync(busy, 0, graph_trips * sizeof(unsigned), stream), "memset busy");
        const uint64_t l0 = launches;
        for (size_t j = 0; j < graph_trips; ++j) launch_trip(busy + j, nullptr);
        per_graph_launches = launches - l0;
        launches = l0;  // counted per graph launch below
        capg.active = false;
        check(cudaStreamEndCapture(stream, &gh.graph), "end capture");
        check(cudaGraphInstantiate(&gh.exec, gh.graph, 0), "graph instantiate");
      };
      capture();
      for (;;) {
        check(cudaGraphLaunch(gh.exec, stream), "graph launch");
        check(cudaMemcpyAsync(mbox, busy + graph_trips - 1, sizeof(unsigned), cudaMemcpyDeviceToHost, stream), "D2H");
        check(cudaMemcpyAsync(mbox + 1, a.next, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream), "D2H");
        check(cudaStreamSynchronize(stream), "tracker trips");
        trips += graph_trips;
        launches += per_graph_launches;
        const unsigned long long nbusy = *reinterpret_cast<unsigned*>(mbox);
        drain_events();
        if (nbusy == 0) break;
        if (maybe_compact(nbusy, mbox[1])) capture();
      }
    }
  }
  unsigned long long work[2] = {0, 0};
  check(cudaMemcpyAsync(work, a.work, sizeof work, cudaMemcpyDeviceToHost, stream), "D2H");
  check(cudaEventRecord(e[2], stream), "event");

  // records back to the caller's host buffers
  std::vector<double> div(count * 4);
  std::vector<uint8_t> divflag(count);
  auto down = [&](void* dst, const void* src, size_t b) {
    if (b) check(cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToHost, stream), "D2H");
  };
  down(out->x, a.rec_x, rec_bytes_x);
  down(out->residual, a.rec_res, count * L * sizeof(double));
  down(out->status, a.rec_status, count);
  down(out->reason, a.rec_reason, count);
  down(out->steps, a.rec_steps, count * 4);
  down(out->newton_iters, a.rec_newton, count * 4);
  down(out->rejections, a.rec_rej, count * 4);
  down(div.data(), a.rec_div, count * 4 * sizeof(double));
  down(divflag.data(), a.rec_divflag, count);
  check(cudaEventRecord(e[3], stream), "event");
  temps.release();
  check(cudaStreamSynchronize(stream), "record download");
  float ms_h2d = 0, ms_k = 0, ms_d2h = 0;
  check(cudaEventElapsedTime(&ms_h2d, e[0], e[1]), "event time");
  check(cudaEventElapsedTime(&ms_k, e[1], e[2]), "event time");
  check(cudaEventElapsedTime(&ms_d2h, e[2], e[3]), "event time");

  // terminal divergence classification: m_est = log(growth) / log(shrink) with the host libm
  // (tracker.cpp:429-431); path ids of the shard's records
  const uint64_t blk = a.shard_block;
  uint64_t newton_sum = 0;
  for (uint64_t i = 0; i < count; ++i) {
    out->path_id[i] = lo + ((i / blk) * a.shard_n + a.shard_r) * blk + i % blk;
    newton_sum += out->newton_iters[i];
    if (!divflag[i]) continue;
    const double first = div[i * 4 + 0], last = div[i * 4 + 1], uf = div[i * 4 + 2], ul = div[i * 4 + 3];
    const double m_est = std::log(last / first) / std::log(uf / ul);
    if (last >= 10.0 && m_est >= 0.05) out->reason[i] = PP_REASON_DIVERGED;
  }
  out->count = count;
  if (stats) {
    stats->paths = count;
    stats->batches = 1;
    stats->total_rounds = trips;
    stats->newton_iters = newton_sum;
    stats->device_ms = ms_k;
    stats->h2d_ms = ms_h2d;
    stats->d2h_ms = ms_d2h;
    stats->h2d_bytes = h2d;
    stats->d2h_bytes = rec_bytes_x + count * (L * 8 + 2 + 12 + 33);
    stats->slots = static_cast<uint32_t>(S);
    stats->kernel_launches = static_cast<uint32_t>(launches);
    stats->evals = work[0];
    stats->solves = work[1];
    stats->eval_ms = kms[0];
    stats->lsq_ms = kms[1];
    stats->step_ms = kms[2];
    stats->events = n_events;
    stats->wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
  }
  (void)compactions;
}

// ---------------------------------------------------------------------------------------------
// kernel-level parity entry points (host <-> planar transposition happens here)
// ---------------------------------------------------------------------------------------------
namespace {
// the planar accessors form offsets in 32 bits (track_impl.cuh, Planar::at): every planar array of
// a kernel-level call must hold fewer than 2^32 doubles (callers chunk larger batches)
void check_planar_size(size_t doubles, const char* what) {
  if (doubles >= (static_cast<size_t>(1) << 32))
    throw InvalidArgument(std::string(what) + ": batch too large (a planar array would exceed 2^32 doubles)");
}

// user layout [item][elem][2L]  <->  planar [elem][plane][item]
void to_planar(const double* src, double* dst, size_t items, size_t elems, size_t w) {
  for (size_t i = 0; i < items; ++i)
    for (size_t e = 0; e < elems; ++e)
      for (size_t p = 0; p < w; ++p) dst[(e * w + p) * items + i] = src[(i * elems + e) * w + p];
}
void from_planar(const double* src, double* dst, size_t items, size_t elems, size_t w) {
  for (size_t i = 0; i < items; ++i)
    for (size_t e = 0; e < elems; ++e)
      for (size_t p = 0; p < w; ++p) dst[(i * elems + e) * w + p] = src[(e * w + p) * items + i];
}
}  // namespace

void device_eval(const Plan& plan, DevicePlan* dp, uint32_t batch, const double* points,
                 const double* t, double* sys, double* jac, int device) {
  if (batch == 0) return;
  DeviceGuard g(device);
  const uint32_t n = plan.dim, np = plan.n_polys, L = plan.L, w = 2 * L;
  const dev::Variant* var = pick_variant(plan.prec, n, plan.max_k);
  if (var == nullptr) throw InvalidArgument("system beyond the compiled kernels");
  check_planar_size(static_cast<size_t>(np) * n * w * batch, "pp_eval_batch");
  std::vector<double> xp(static_cast<size_t>(batch) * n * w), tp(static_cast<size_t>(batch) * L);
  to_planar(points, xp.data(), batch, n, w);
  to_planar(t, tp.data(), batch, 1, L);
  DevBuf<double> dx(xp);
  DevBuf<double> dt(tp);
  DevBuf<double> ds(static_cast<size_t>(batch) * np * w);
  DevBuf<double> dj(static_cast<size_t>(batch) * np * n * w);
  dev::EvalArgs a{};
  a.plan = plan_args(plan, dp);
  a.batch = batch;
  a.x = dx.p;
  a.t = dt.p;
  a.sys = ds.p;
  a.jac = dj.p;
  int block = 128;
  while (block > 32 && static_cast<size_t>(block) * 2 * n * w * sizeof(double) > 200 * 1024) block /= 2;
  const size_t smem = static_cast<size_t>(block) * 2 * n * w * sizeof(double);
  ensure_smem(var->eval, smem, device);
  void* args[] = {&a};
  check(cudaLaunchKernel(var->eval, dim3((batch + block - 1) / block), dim3(block), args, smem, 0), "launch eval");
  check(cudaDeviceSynchronize(), "eval kernel");
  std::vector<double> hs(static_cast<size_t>(batch) * np * w), hj(static_cast<size_t>(batch) * np * n * w);
  check(cudaMemcpy(hs.data(), ds.p, hs.size() * 8, cudaMemcpyDeviceToHost), "D2H");
  check(cudaMemcpy(hj.data(), dj.p, hj.size() * 8, cudaMemcpyDeviceToHost), "D2H");
  from_planar(hs.data(), sys, batch, np, w);
  if (jac) {
    // planar element v*np + p  ->  user row p*n + v
    for (size_t i = 0; i < batch; ++i)
      for (size_t p = 0; p < np; ++p)
        for (size_t v = 0; v < n; ++v)
          for (size_t q = 0; q < w; ++q)
            jac[((i * np + p) * n + v) * w + q] = hj[((v * np + p) * w + q) * batch + i];
  }
}

// bench-eval (polypath_main.cpp:284-362) on the device: the evaluation kernel over `batch` points
// given in the reference's planar layout (points [v][plane][batch], t [plane][batch]), timed with
// CUDA events over `reps` launches after one warm-up launch; sys [p][plane][batch] and the
// Jacobian in the reference's row order [p*dim + v][plane][batch] are returned for the checksum.
double device_bench_eval(const Plan& plan, DevicePlan* dp, uint32_t batch, const double* xp, const double* tp,
                         uint32_t reps, double* sys, double* jac, int device) {
  DeviceGuard g(device);
  const uint32_t n = plan.dim, np = plan.n_polys, L = plan.L, w = 2 * L;
  const dev::Variant* var = pick_variant(plan.prec, n, plan.max_k);
  if (var == nullptr) throw InvalidArgument("system beyond the compiled kernels");
  check_planar_size(static_cast<size_t>(np) * n * w * batch, "pp_bench_eval");
  std::vector<double> xv(xp, xp + static_cast<size_t>(batch) * n * w), tv(tp, tp + static_cast<size_t>(batch) * L);
  DevBuf<double> dx(xv);
  DevBuf<double> dt(tv);
  DevBuf<double> ds(static_cast<size_t>(batch) * np * w);
  DevBuf<double> dj(static_cast<size_t>(batch) * np * n * w);
  dev::EvalArgs a{};
  a.plan = plan_args(plan, dp);
  a.batch = batch;
  a.x = dx.p;
  a.t = dt.p;
  a.sys = ds.p;
  a.jac = dj.p;
  int block = 128;
  while (block > 32 && static_cast<size_t>(block) * 2 * n * w * sizeof(double) > 200 * 1024) block /= 2;
  const size_t smem = static_cast<size_t>(block) * 2 * n * w * sizeof(double);
  ensure_smem(var->eval, smem, device);
  void* args[] = {&a};
  const dim3 grid((batch + block - 1) / block);
  check(cudaLaunchKernel(var->eval, grid, dim3(block), args, smem, 0), "launch eval");  // warm-up
  EvPair ev;
  check(cudaEventRecord(ev.e0, 0), "event");
  for (uint32_t r = 0; r < std::max<uint32_t>(reps, 1); ++r)
    check(cudaLaunchKernel(var->eval, grid, dim3(block), args, smem, 0), "launch eval");
  check(cudaEventRecord(ev.e1, 0), "event");
  check(cudaEventSynchronize(ev.e1), "eval kernel");
  float ms = 0;
  check(cudaEventElapsedTime(&ms, ev.e0, ev.e1), "event time");
  // eval_kernel returns H (not -H) in sys
  check(cudaMemcpy(sys, ds.p, static_cast<size_t>(batch) * np * w * 8, cudaMemcpyDeviceToHost), "D2H");
  std::vector<double> hj(static_cast<size_t>(batch) * np * n * w);
  check(cudaMemcpy(hj.data(), dj.p, hj.size() * 8, cudaMemcpyDeviceToHost), "D2H");
  for (size_t p = 0; p < np; ++p)
    for (size_t v = 0; v < n; ++v)
      std::memcpy(jac + (p * n + v) * w * batch, hj.data() + (v * np + p) * w * batch, w * batch * sizeof(double));
  return ms / std::max<uint32_t>(reps, 1);
}

// the corrector alone for `batch` (t, x) pairs (layouts of pp_test_newton)
void device_newton(const Plan& plan, DevicePlan* dp, const pp_track_config& cfg, uint32_t batch, const double* t,
                   double* x, uint32_t* iters, uint8_t* corrected, uint8_t* singular, int device) {
  if (batch == 0) return;
  DeviceGuard g(device);
  const uint32_t n = plan.dim, L = plan.L, w = 2 * L;
  const dev::Variant* var = pick_variant(plan.prec, n, plan.max_k);
  if (var == nullptr) throw InvalidArgument("system beyond the compiled kernels");
  check_planar_size(static_cast<size_t>(n) * n * w * batch, "pp_test_newton");
  std::vector<double> xp(static_cast<size_t>(batch) * n * w), tp(static_cast<size_t>(batch) * L);
  to_planar(x, xp.data(), batch, n, w);
  to_planar(t, tp.data(), batch, 1, L);
  DevBuf<double> dx(xp), dt(tp), dj(static_cast<size_t>(batch) * n * n * w),
      dr(static_cast<size_t>(batch) * n * (n + 1) / 2 * w), db(static_cast<size_t>(batch) * n * w),
      dy(static_cast<size_t>(batch) * n * w);
  DevBuf<uint32_t> di(batch);
  DevBuf<uint8_t> dc(batch), ds(batch);
  dev::NewtonArgs a{};
  a.plan = plan_args(plan, dp);
  a.batch = batch;
  a.max_newton = cfg.max_newton;
  a.rtol = cfg.residual_tol;
  a.utol = cfg.update_tol;
  a.rank_tol = default_rank_tol(plan.prec);
  a.x = dx.p;
  a.t = dt.p;
  a.J = dj.p;
  a.Rm = dr.p;
  a.B = db.p;
  a.Y = dy.p;
  a.iters = di.p;
  a.corrected = dc.p;
  a.singular = ds.p;
  int block = 128;
  while (block > 32 && static_cast<size_t>(block) * 3 * n * w * sizeof(double) > 200 * 1024) block /= 2;
  const size_t smem = static_cast<size_t>(block) * 3 * n * w * sizeof(double);
  ensure_smem(var->newton, smem, device);
  void* args[] = {&a};
  check(cudaLaunchKernel(var->newton, dim3((batch + block - 1) / block), dim3(block), args, smem, 0), "launch newton");
  check(cudaDeviceSynchronize(), "newton kernel");
  check(cudaMemcpy(xp.data(), dx.p, xp.size() * 8, cudaMemcpyDeviceToHost), "D2H");
  check(cudaMemcpy(iters, di.p, batch * 4, cudaMemcpyDeviceToHost), "D2H");
  check(cudaMemcpy(corrected, dc.p, batch, cudaMemcpyDeviceToHost), "D2H");
  check(cudaMemcpy(singular, ds.p, batch, cudaMemcpyDeviceToHost), "D2H");
  from_planar(xp.data(), x, batch, n, w);
}

void device_lsq(int prec, uint32_t m, uint32_t n, uint32_t batch, const double* a, const double* b, double* x,
                uint8_t* ok, double* q_out, double* r_out, int device) {
  if (batch == 0) return;
  DeviceGuard g(device);
  const uint32_t L = prec == 0 ? 1 : (prec == 1 ? 2 : 4), w = 2 * L;
  const dev::Variant* var = pick_variant(prec, std::max(m, n), 2);
  if (var == nullptr) throw InvalidArgument("least-squares size beyond the compiled kernels");
  check_planar_size(static_cast<size_t>(m) * n * w * batch, "pp_lsq_batch");
  const size_t nr = static_cast<size_t>(n) * (n + 1) / 2;
  std::vector<double> ap(static_cast<size_t>(batch) * m * n * w), bp(static_cast<size_t>(batch) * m * w);
  to_planar(a, ap.data(), batch, static_cast<size_t>(m) * n, w);
  to_planar(b, bp.data(), batch, m, w);
  DevBuf<double> da(ap), db(bp), dr(static_cast<size_t>(batch) * nr * w), dy(static_cast<size_t>(batch) * n * w),
      dxv(static_cast<size_t>(batch) * n * w);
  DevBuf<uint8_t> dok(batch);
  dev::LsqArgs args{static_cast<int>(n), static_cast<int>(m), batch, default_rank_tol(prec), da.p, dr.p, db.p, dy.p,
                    dxv.p, dok.p};
  void* pa[] = {&args};
  int block = 128;
  while (block > 32 && static_cast<size_t>(block) * m * w * sizeof(double) > 200 * 1024) block /= 2;
  const size_t smem = static_cast<size_t>(block) * m * w * sizeof(double);
  ensure_smem(var->lsq, smem, device);
  check(cudaLaunchKernel(var->lsq, dim3((batch + block - 1) / block), dim3(block), pa, smem, 0), "launch lsq");
  check(cudaDeviceSynchronize(), "lsq kernel");
  std::vector<double> hx(static_cast<size_t>(batch) * n * w);
  check(cudaMemcpy(hx.data(), dxv.p, hx.size() * 8, cudaMemcpyDeviceToHost), "D2H");
  check(cudaMemcpy(ok, dok.p, batch, cudaMemcpyDeviceToHost), "D2H");
  from_planar(hx.data(), x, batch, n, w);
  if (q_out) {  // Q, column-major m x n per system
    std::vector<double> hq(ap.size());
    check(cudaMemcpy(hq.data(), da.p, hq.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    from_planar(hq.data(), q_out, batch, static_cast<size_t>(m) * n, w);
  }
  if (r_out) {  // R, packed upper triangle: (row j, column i >= j) at j + i(i+1)/2
    std::vector<double> hr(static_cast<size_t>(batch) * nr * w);
    check(cudaMemcpy(hr.data(), dr.p, hr.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    from_planar(hr.data(), r_out, batch, nr, w);
  }
}

}  // namespace pp
