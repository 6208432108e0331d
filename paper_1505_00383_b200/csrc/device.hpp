// device.hpp -- internal interface between the host C ABI (capi.cpp) and the CUDA side.
#pragma once

#include <string>

#include "host.hpp"
#include "pp200.h"

namespace pp {

// Thrown by the CUDA side on any runtime failure; mapped to PP_E_CUDA at the C ABI.
struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Device-resident copy of a plan (SoA tables), built once per homotopy and reused by every call.
struct DevicePlan;
DevicePlan* device_plan_upload(const Plan& plan, int device);
void device_plan_free(DevicePlan* dp);

// block-cyclic shard of a start range (pp_shard); count == 1 is the whole range
struct TrackShard {
  uint64_t index = 0, count = 1, block = 1;
};
uint64_t shard_size(uint64_t lo, uint64_t hi, const TrackShard& sh);

// step-event sink (ProgressSink); fn == nullptr disables events
struct EventSink {
  pp_event_sink fn = nullptr;
  void* user = nullptr;
};

// track_all on the device: the shard's starts of [lo, hi) -> records (host buffers in `out`).
void device_track(const Plan& plan, DevicePlan* dp, const Starts& st, const pp_track_config& cfg,
                  uint64_t lo, uint64_t hi, const TrackShard& shard, const EventSink& sink, int device,
                  pp_records* out, pp_run_stats* stats);

// eval_system_batch on the device (host buffers, layouts of pp_eval_batch)
void device_eval(const Plan& plan, DevicePlan* dp, uint32_t batch, const double* points,
                 const double* t, double* sys, double* jac, int device);

// bench-eval on the device (reference planar layouts); returns ms per evaluation launch
double device_bench_eval(const Plan& plan, DevicePlan* dp, uint32_t batch, const double* xp, const double* tp,
                         uint32_t reps, double* sys, double* jac, int device);

// batched least_squares_solve / mgs_qr for m x n systems (layouts of pp_lsq_batch_mn)
void device_lsq(int prec, uint32_t m, uint32_t n, uint32_t batch, const double* a, const double* b, double* x,
                uint8_t* ok, double* q_out, double* r_out, int device);

// the corrector alone for `batch` (t, x) pairs (pp_test_newton)
void device_newton(const Plan& plan, DevicePlan* dp, const pp_track_config& cfg, uint32_t batch, const double* t,
                   double* x, uint32_t* iters, uint8_t* corrected, uint8_t* singular, int device);

// rank tolerance of the reference's least_squares_solve default (linalg.hpp:44-52)
inline double default_rank_tol(int prec) { return prec == 0 ? 1e-8 : (prec == 1 ? 1e-16 : 1e-32); }

// largest dimension / monomial support the compiled kernels cover
bool device_supports(uint32_t n, uint32_t max_k);

// CUDA devices visible (0 without a usable driver)
int device_count();

// context, per-thread resources and kernel modules of a device, created ahead of the first call
void device_init(int device);

// measured FP64 pipe operations per second (DFMA microbenchmark)
double device_fp64_peak(int device);

}  // namespace pp
