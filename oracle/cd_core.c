/*
 * cd_core.c — ORACLE / TEST INFRASTRUCTURE ONLY (never the product path).
 *
 * Plain-C restatement of the reference's numba core `_cd_sweeps_jit`
 * (reference pkg/src/fieldfit/elastic_net.py:113-161): cyclic coordinate
 * descent in residual form over a Fortran-ordered (n, m) design matrix.
 * Compiled with -O2 -ffp-contract=off so every `a*b + c` is a separate
 * multiply and add, exactly as numba (fastmath=False) evaluates it; loops are
 * sequential in the reference's order, so results are bit-identical to the
 * reference when fed identical inputs (pinned in tests/test_oracle_pins.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
 * arm may load this library.
 */
#include <math.h>
#include <stdint.h>

/* returns sweeps; *converged set to 0/1.  Mutates beta, r, history. */
int64_t oracle_cd_sweeps(const double* W, int64_t n, int64_t m, const double* col_sq,
                         const double* denom, double lam1, double lam2, double tol,
                         int64_t max_iters, double* beta, double* r, double* history,
                         int32_t* converged) {
  int64_t sweeps = 0;
  *converged = 0;
  for (int64_t s = 0; s < max_iters; ++s) {
    double max_delta = 0.0;
    for (int64_t j = 0; j < m; ++j) {
      const double* col = W + j * n; /* Fortran order: column j contiguous */
      double b_old = beta[j];
      double z = col_sq[j] * b_old;
      for (int64_t i = 0; i < n; ++i) z += col[i] * r[i];
      double b_new;
      if (denom[j] > 0.0) {
        double mag = fabs(z) - lam1;
        if (mag < 0.0) mag = 0.0;
        b_new = (z >= 0.0 ? mag : -mag) / denom[j];
      } else {
        b_new = 0.0;
      }
      if (b_new != b_old) {
        double d = b_new - b_old;
        for (int64_t i = 0; i < n; ++i) r[i] -= d * col[i];
        beta[j] = b_new;
        if (fabs(d) > max_delta) max_delta = fabs(d);
      }
    }
    double rss = 0.0;
    for (int64_t i = 0; i < n; ++i) rss += r[i] * r[i];
    double l1 = 0.0, l2 = 0.0, max_abs = 0.0;
    for (int64_t j = 0; j < m; ++j) {
      double a = fabs(beta[j]);
      l1 += a;
      l2 += beta[j] * beta[j];
      if (a > max_abs) max_abs = a;
    }
    history[s] = 0.5 * rss + lam1 * l1 + 0.5 * lam2 * l2;
    sweeps = s + 1;
    if (max_delta <= tol * (max_abs > 1.0 ? max_abs : 1.0)) {
      *converged = 1;
      break;
    }
  }
  return sweeps;
}
