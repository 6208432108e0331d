/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.  A plain-C restatement of the reference tracker's
 * algorithm (polypath, /root/reference/proj) for ONE path at a time, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the checker.  The product never
 * links, imports or calls it.
 *
 * Pinned against the reference itself: tests/test_oracle.py compares it bit for bit with the
 * reference library built from its own sources (oracle/_ref, oracle/Makefile) and with the
 * committed golden fixtures in tests/golden/.
 *
 * Values at level L (1 = double, 2 = double-double, 4 = quad-double) are arrays of L doubles;
 * complex values are [re limbs..., im limbs...].
 */
#ifndef PP_ORACLE_H
#define PP_ORACLE_H

#include <stdint.h>

/* merged plan (reference EvalPlan, evaldiff.hpp:80-94): term i has poly term_info[4i],
 * k = term_info[4i+1] variables at pos[term_info[4i+2] + j] = var | (exponent << 16);
 * coeff[i] = (c_start, c_target), 2L doubles each */
typedef struct oracle_plan {
  int L;
  int dim, n_polys, n_terms;
  const int32_t* term_info;
  const uint32_t* pos;
  const double* coeff;
} oracle_plan;

/* TrackConfig (tracker.hpp:29-46) */
typedef struct oracle_cfg {
  double residual_tol, update_tol;
  int max_newton, expand_after;
  double h_init, h_min, h_max, expand, contract, divergence_bound;
  uint32_t max_steps;
} oracle_cfg;

/* eval_single: H(x, t) and the row-major Jacobian (row = poly*dim + var) */
int oracle_eval(const oracle_plan* p, const double* x, const double* t, double* sys, double* jac);
/* least_squares_solve: a column-major n x n (element col*n + row), returns 1 ok / 0 rank-deficient */
int oracle_lsq(int L, int n, const double* a, const double* b, double* x);
/* one path of track_all from start x0: writes the endpoint (xacc), residual (L doubles) and
 * info = {status, reason, steps, newton_iters, rejections} */
int oracle_track_path(const oracle_plan* p, const oracle_cfg* c, const double* x0, double* x_out,
                      double* resid_out, int32_t* info);
/* scalar arithmetic at a level (op codes of pp200_testing.h) */
int oracle_arith(int L, int op, const double* a, const double* b, double* out);

#endif
