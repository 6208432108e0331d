/*
 * pp200_testing.h -- test hooks exported by libpp200.so in addition to pp200.h.  Not part of the
 * drop-in boundary; used by tests/ to compare the host arithmetic, decimal I/O and plan tables
 * with the reference build bit for bit.
 */
#ifndef PP200_TESTING_H
#define PP200_TESTING_H

#include <stddef.h>
#include <stdint.h>

#include "pp200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* op: 0 add, 1 sub, 2 mul, 3 mul by double b[0], 4 div, 5 sqrt, 6 compare, 7 to_double,
 * 8 complex mul, 9 complex div (Smith), 10 complex modulus.  Operands are limb arrays. */
int pp_test_arith(int prec, int op, const double* a, const double* b, double* out);
/* parse_decimal at a level (xprec_io.cpp:121-193) */
int pp_test_parse_decimal(int prec, const char* s, double* out);
/* to_decimal at a level (xprec_io.cpp:31-108, 198-212) */
int pp_test_to_decimal(int prec, const double* in, char* buf, size_t cap);
/* per-term (c_start, c_target) coefficient limbs of a homotopy's plan */
int pp_test_plan_coeffs(const pp_homotopy* h, double* out, size_t cap);
/* plan tables: which = 0 term_slot, 1 acc_off, 2 acc_idx (warp-per-path accumulation lists),
 * 3 pos, 4 term_info; *count = entries (PP_E_CAPACITY when cap is too small) */
int pp_test_plan_tables(const pp_homotopy* h, int which, uint32_t* out, size_t cap, size_t* count);
/* measured FP64 pipe throughput of a device (DFMA ops/s), the roofline denominator */
int pp_fp64_peak(int device, double* ops_per_s);
/* n doubles formatted as the JSON-lines records print them (nlohmann::json 3.11's dump()),
 * newline-separated; *needed = bytes including the NUL (PP_E_CAPACITY when cap is too small) */
int pp_test_json_doubles(const double* v, size_t n, char* buf, size_t cap, size_t* needed);
/* The corrector alone, as the reference's tests drive it through PathBatch::set_prediction and
 * newton_correct (tracker.hpp:135-136, tracker.cpp:216-274): for each of `batch` pairs (t [L], x
 * [dim][2L]) run up to cfg->max_newton Newton iterations at that t on the device.  Outputs the
 * iterations performed (last_iterations), whether the residual / update test certified the step
 * (last_corrected), whether a solve was rank-deficient, and the last iterate (in place in x). */
int pp_test_newton(const pp_homotopy* h, const pp_track_config* cfg, uint32_t batch, const double* t, double* x,
                   uint32_t* iters, uint8_t* corrected, uint8_t* singular, int device);
/* [mon_steps, cmul_steps, jac_terms, jac_scaled, n_base] of a homotopy's plan */
int pp_homotopy_counts(const pp_homotopy* h, uint64_t* counts);

#ifdef __cplusplus
}
#endif

#endif
