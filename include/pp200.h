/*
 * pp200.h -- C ABI of the B200-native many-path homotopy tracker.
 *
 * This is the drop-in boundary for the reference's hot path
 *   template<class R> SolutionSet<R> track_all(const HomotopyInstance<R>&,
 *       const StartData<R>&, const TrackConfig&, ProgressSink*, uint64_t lo, uint64_t hi)
 *   (reference: proj/include/polypath/tracker.hpp:166-170, impl proj/src/tracker.cpp:511-540)
 * and of the host calls that feed it (system parsing, homotopy construction, start data).
 * Every entry point takes plain pointers and sizes; no C++ or torch types cross it.
 *
 * Precision is a runtime tag (reference: xprec.hpp:547 `enum class Precision {d, dd, qd}`).
 * A value at precision R is stored as L = 1/2/4 binary64 limbs, most significant first;
 * a complex value is [re limbs..., im limbs...] (2L doubles), the order of the reference's
 * PlanarBlock planes (evaldiff.hpp:114-172).
 *
 * Errors: 0 = success; negative codes below.  PP_E_INVALID corresponds to the reference's
 * std::invalid_argument (TrackConfig::validate, tracker.cpp:40-49; empty start set,
 * tracker.cpp:516; dimension checks, homotopy.cpp:9-13).  PP_E_PARSE corresponds to
 * polypath::ParseError (polysys.hpp:60-65); its line/column are in pp_last_error().
 * Per-path failures are data (status/reason), never error codes (tracker.hpp:16-25).
 * There is no CPU fallback: if no CUDA device is usable, device entry points return PP_E_CUDA.
 */
#ifndef PP200_H
#define PP200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* precision tags (xprec.hpp:547) */
enum { PP_D = 0, PP_DD = 1, PP_QD = 2 };

/* error codes */
enum {
  PP_OK = 0,
  PP_E_INVALID = -1,  /* std::invalid_argument in the reference */
  PP_E_PARSE = -2,    /* polypath::ParseError */
  PP_E_CUDA = -3,     /* CUDA runtime failure / no device */
  PP_E_NOMEM = -4,
  PP_E_CAPACITY = -5, /* caller buffer too small */
  PP_E_DOMAIN = -6    /* std::domain_error (division by zero in xprec/complex) */
};

/* PathStatus (tracker.hpp:16) */
enum { PP_FAILED = -1, PP_ACTIVE = 0, PP_SUCCESS = 1 };

/* FailReason (tracker.hpp:18-25) */
enum {
  PP_REASON_NONE = 0,
  PP_REASON_DIVERGED = 1,
  PP_REASON_STEP_UNDERFLOW = 2,
  PP_REASON_MAX_STEPS = 3,
  PP_REASON_SINGULAR = 4,
  PP_REASON_NO_CERTIFICATE = 5
};

/* TrackConfig (tracker.hpp:29-46); field meaning and defaults identical. */
typedef struct pp_track_config {
  double residual_tol;
  double update_tol;
  int32_t max_newton;
  int32_t expand_after;
  double h_init;
  double h_min;
  double h_max;
  double expand;
  double contract;
  double divergence_bound;
  uint32_t max_steps;
  uint32_t batch;   /* reference cohort width; the device ignores it (persistent refill) */
  uint32_t workers; /* reference CPU workers; the device ignores it */
  uint32_t reserved;
} pp_track_config;

/*
 * Output records: SolutionSet<R>::paths (tracker.hpp:73-94) as caller-owned SoA host buffers.
 * Record i belongs to start index lo+i, so the set is sorted by path_id as in
 * tracker.cpp:537-538.  x is [record][var][2L] doubles, residual is [record][L].
 */
typedef struct pp_records {
  uint64_t capacity; /* records the buffers can hold (>= hi-lo) */
  uint64_t count;    /* out: records written */
  uint64_t* path_id;
  int8_t* status;
  uint8_t* reason;
  uint32_t* steps;
  uint32_t* newton_iters;
  uint32_t* rejections;
  double* x;
  double* residual;
} pp_records;

/* Run statistics (SolutionSet::batches/total_rounds, tracker.hpp:89-94, plus device timing) */
typedef struct pp_run_stats {
  uint64_t paths;        /* terminal paths produced */
  uint64_t batches;      /* device launches (the reference's cohorts) */
  uint64_t total_rounds; /* loop trips of the slowest device slot */
  uint64_t newton_iters; /* sum over paths, corrector iterations */
  double device_ms;      /* tracking kernel time (CUDA events) */
  double h2d_ms;         /* host->device staging */
  double d2h_ms;         /* device->host record copy */
  double wall_ms;        /* whole call */
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  uint32_t slots;        /* concurrent path slots on the device */
  uint32_t kernel_launches;
  uint64_t evals;        /* H/Jacobian evaluations performed (corrector + refinement + final) */
  uint64_t solves;       /* least-squares solves performed (corrector + refinement) */
  double eval_ms;        /* per-kernel device time; filled only when PP200_KERNEL_TIMING=1 */
  double lsq_ms;
  double step_ms;
  uint64_t events;       /* step events handed to the sink (pp_track_all_ex) */
} pp_run_stats;

typedef struct pp_system pp_system;     /* PolySystem (polysys.hpp:41-51) */
typedef struct pp_starts pp_starts;     /* StartData<R> (homotopy.hpp:38-49) */
typedef struct pp_homotopy pp_homotopy; /* HomotopyInstance<R> + device plan (homotopy.hpp:16-22) */

const char* pp_version(void);
/* message of the last failing call on this thread ("" if none) */
const char* pp_last_error(void);
/* number of binary64 limbs of a precision tag, 0 if the tag is invalid */
int pp_limbs(int prec);

/* ---- systems: polysys.hpp:67-79 (parse_system, print_system, cyclic_system, system_stats) ---- */
int pp_system_parse(const char* text, size_t len, pp_system** out);
int pp_system_cyclic(uint32_t n, pp_system** out);
/* PolySystem from its terms (polysys.hpp:21-50) without a text round trip: term_count[p] terms in
 * polynomial p; term t has n_factors[t] (variable, exponent) pairs in `factors` (concatenated, sorted
 * by variable, exponents >= 1) and the coefficient coeff[8t .. 8t+7] = Cplx<QD> (re limbs, im limbs).
 * The reference host shim passes the reference's in-memory systems through this entry point. */
int pp_system_from_terms(uint32_t dim, uint32_t n_polys, const uint32_t* term_count, const uint32_t* n_factors,
                         const uint32_t* factors, const double* coeff, pp_system** out);
/* CUDA devices visible to the library (0 without a usable driver) */
int pp_device_count(void);
/* create the CUDA context of `device`, the calling thread's stream and workspace context, and load
 * the tracking kernels, so that the first pp_track_all on this thread does not pay for them
 * (about 1.8 s on a fresh B200 process); optional */
int pp_device_init(int device);
/* writes a NUL-terminated text form; *needed = bytes required including the NUL */
int pp_system_print(const pp_system* s, char* buf, size_t cap, size_t* needed);
int pp_system_stats(const pp_system* s, uint32_t* dim, uint32_t* n_polys, uint64_t* n_monomials,
                    uint64_t* total_degree, int* total_degree_overflow);
/* per-polynomial total degrees, n_polys entries */
int pp_system_degrees(const pp_system* s, uint32_t* degrees);
void pp_system_free(pp_system* s);

/* ---- homotopy.hpp:24-68 ---- */
/* random_gamma(seed) (homotopy.cpp:34-40) */
void pp_random_gamma(uint64_t seed, double* re, double* im);
/* total_degree_start<R>(f) (homotopy.cpp:87-113): start system g and lazily indexed starts */
int pp_total_degree_start(const pp_system* f, int prec, pp_system** g_out, pp_starts** out);
/* load_start_data<R>(g, parse_solutions(text), start_tol) (homotopy.cpp:115-140, polysys.cpp:381-425).
 * The residual screening runs on the device.  Rejected candidates (0-based index and residual) are
 * written to rejected_idx / rejected_resid up to rejected_cap entries; *n_rejected is the total. */
int pp_load_start_data(const pp_system* g, int prec, const char* text, size_t len, double start_tol,
                       int device, pp_starts** out, uint64_t* rejected_idx,
                       double* rejected_resid, uint64_t rejected_cap, uint64_t* n_rejected);
/* explicit start list, [count][dim][2L] doubles (StartProvenance::file) */
int pp_starts_explicit(int prec, uint32_t dim, uint64_t count, const double* x, pp_starts** out);
/* StartData<R> in total-degree mode from its own tables (homotopy.hpp:38-49): degrees[dim] and
 * the per-variable root tables concatenated, sum(degrees) complex values of 2L doubles.
 * Index enumeration is StartData::solution's (homotopy.cpp:73-85, last variable fastest). */
int pp_starts_roots(int prec, uint32_t dim, const uint32_t* degrees, const double* roots, pp_starts** out);
uint64_t pp_starts_count(const pp_starts* s);
/* StartData::solution(index) (homotopy.cpp:73-85), dim×2L doubles */
int pp_starts_solution(const pp_starts* s, uint64_t index, double* x);
void pp_starts_free(pp_starts* s);

/* make_homotopy<R>(f, g, gamma) (homotopy.cpp:7-20); gamma is 2L doubles (re limbs, im limbs) */
int pp_make_homotopy(const pp_system* f, const pp_system* g, int prec, const double* gamma,
                     pp_homotopy** out);
/* plan geometry (EvalPlan, evaldiff.hpp:80-94) */
int pp_homotopy_info(const pp_homotopy* h, uint32_t* dim, uint32_t* n_polys, uint32_t* n_terms,
                     uint32_t* mon_rows, uint32_t* max_k, uint64_t* posprod_muls);
void pp_homotopy_free(pp_homotopy* h);

/* ---- tracker.hpp:29-46 ---- */
void pp_track_config_defaults(int prec, pp_track_config* cfg); /* TrackConfig::defaults */
int pp_track_config_validate(const pp_track_config* cfg);      /* TrackConfig::validate */

/*
 * track_all<R> (tracker.hpp:166-170): tracks starts [lo, min(count, hi)) on CUDA device `device`
 * and writes one record per start into `out`.  Returns PP_E_INVALID for a bad config or an empty
 * start set, exactly where the reference throws.  stats may be NULL.
 */
int pp_track_all(const pp_homotopy* h, const pp_starts* s, const pp_track_config* cfg,
                 uint64_t lo, uint64_t hi, int device, pp_records* out, pp_run_stats* stats);

/*
 * StepEvent (tracker.hpp:62-69) and ProgressSink (tracker.hpp:70).  The reference invokes the sink
 * once per active path and lockstep round inside step_control_all (tracker.cpp:312-315), after the
 * step decision: t and h are the new values, newton_iters the corrector iterations of this step,
 * status the path's status before this round's check (always PP_ACTIVE), accepted the decision.
 * The device appends the same records to an event ring; the host hands them to the sink in
 * batches, on the calling thread, while tracking proceeds.  Events of one path arrive in the
 * order the reference emits them; events of different paths interleave in device order.
 */
typedef struct pp_step_event {
  uint64_t path_id;
  double t;
  double h;
  uint32_t newton_iters;
  int8_t status;
  uint8_t accepted;
  uint8_t reserved[2];
} pp_step_event;
typedef void (*pp_event_sink)(const pp_step_event* events, uint64_t count, void* user);

/*
 * Block-cyclic shard of a start range (multi-GPU): start index i of [lo, hi) belongs to
 * shard ((i - lo) / block) % count.  Interleaving blocks over the shards evens out the per-shard
 * cost, which varies strongly with the start index.  A NULL shard (or count 1) is the whole range.
 */
typedef struct pp_shard {
  uint32_t index; /* this shard, 0 <= index < count */
  uint32_t count; /* number of shards */
  uint64_t block; /* consecutive start indices per block (>= 1) */
} pp_shard;

/* number of start indices of [lo, hi) in shard `shard` (hi already clamped to the start count) */
uint64_t pp_shard_size(uint64_t lo, uint64_t hi, const pp_shard* shard);

/*
 * track_all with the reference's optional arguments: `sink` (NULL = none) receives the step
 * events (ProgressSink, tracker.hpp:166-170), and `shard` (NULL = all) restricts the call to one
 * block-cyclic shard of [lo, min(count, hi)).  Records are written for the shard's start indices
 * in increasing order (path_id carries the index).  pp_track_all(h, s, cfg, lo, hi, dev, out, st)
 * equals pp_track_all_ex(h, s, cfg, lo, hi, NULL, NULL, NULL, dev, out, st).
 */
int pp_track_all_ex(const pp_homotopy* h, const pp_starts* s, const pp_track_config* cfg,
                    uint64_t lo, uint64_t hi, const pp_shard* shard, pp_event_sink sink, void* sink_user,
                    int device, pp_records* out, pp_run_stats* stats);

/*
 * eval_system_batch (evaldiff.hpp:228-230) on the device for `batch` points:
 * points [batch][dim][2L], t [batch][L] -> sys [batch][n_polys][2L], jac [batch][n_polys*dim][2L]
 * (row = poly*dim + var, evaldiff.hpp:181).  jac may be NULL.
 */
int pp_eval_batch(const pp_homotopy* h, uint32_t batch, const double* points, const double* t,
                  double* sys, double* jac, int device);

/*
 * least_squares_solve (linalg.hpp:110-125) for `batch` independent n×n complex systems on the
 * device: a [batch][col][row][2L] (column-major, as DenseMatrix), b [batch][n][2L] ->
 * x [batch][n][2L]; ok[i] = 0 where the reference returns false (rank deficiency).
 */
int pp_lsq_batch(int prec, uint32_t n, uint32_t batch, const double* a, const double* b,
                 double* x, uint8_t* ok, int device);
/*
 * The same for m x n systems (m >= n), as the reference's least_squares_solve and mgs_qr take them
 * (linalg.hpp:79-125): a [batch][col][row][2L] with m rows, b [batch][m][2L]; optionally the
 * factors: q [batch][col][row][2L] (Q, m x n column-major) and r [batch][n(n+1)/2][2L] (R packed by
 * columns: row j, column i >= j at j + i(i+1)/2).  q and r may be NULL.
 */
int pp_lsq_batch_mn(int prec, uint32_t m, uint32_t n, uint32_t batch, const double* a, const double* b,
                    double* x, uint8_t* ok, double* q, double* r, int device);

/*
 * Output records as the reference CLI writes them (polypath_main.cpp:125-189):
 * one JSON "solution" line per record (coordinates as full-precision decimal strings, to_decimal
 * of xprec_io.cpp:31-108), then one "summary" line.  gamma is 2L doubles.  Two-call pattern:
 * returns PP_E_CAPACITY with *needed = bytes required (including the NUL) when buf is too small.
 */
int pp_solutions_jsonl(const pp_records* rec, int prec, uint32_t dim, const double* gamma, uint64_t seed,
                       const char* command, double wall_ms, uint64_t batches, uint64_t rounds, char* buf,
                       size_t cap, size_t* needed);
/*
 * bench-eval (polypath_main.cpp:284-362): `batch` points and t drawn from the
 * CLI's splitmix64 stream for `seed`, one evaluation of H and dH/dx per point on the device,
 * timed over `reps` launches after a warm-up (ms = device time per batch evaluation), and the
 * CLI's FNV-1a checksum of sys then jac in the reference's planar workspace layout.
 */
int pp_bench_eval(const pp_homotopy* h, uint64_t seed, uint32_t batch, uint32_t reps, int device, double* ms,
                  uint64_t* checksum);
/* to_decimal of one level value (xprec_io.cpp:31-108, 198-212): 17 / 32 / 64 significant digits */
int pp_to_decimal(int prec, const double* limbs, char* buf, size_t cap);

#ifdef __cplusplus
}
#endif

#endif /* PP200_H */
