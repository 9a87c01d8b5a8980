/* trisolve.c -- CPU oracle helper (TEST INFRASTRUCTURE ONLY; see oracle/solve.py header).
 *
 * Gauss-Seidel sweeps of the reference (smoothers.py:178-190): the forward sweep solves
 * tril(A) x = b, the backward sweep tril(A)^T x = b, in the natural free-DoF order.  The
 * reference factors tril(A) with SuperLU (permc_spec NATURAL, diag_pivot_thresh 0,
 * SymmetricMode): L = tril(A) diag(A)^-1 (unit), U = diag(A), natural perm_r / perm_c
 * (measured), so its solve is plain substitution.  This file restates that
 * substitution row by row,
 *     forward   x_i = (b_i - sum_{j<i} a_ij x_j) / a_ii,   i = 0 .. n-1
 *     backward  x_i = (b_i - sum_{j>i} a_ji x_j) / a_ii,   i = n-1 .. 0
 * (a_ji = a_ij up to rounding: A is symmetric, assembly.py:611-613), for the sizes where
 * SciPy's splu(tril(A)) does not fit (cfg4 p = 8, cfg5 at full size: 310M / 727M nonzeros).
 * It agrees with SuperLU's supernodal column substitution to rounding (tests/test_oracle.py
 * pins it against splu on every golden configuration).
 *
 * Input is the full CSR of A (int64 row pointers, int32 sorted column indices).  Built by
 * oracle/Makefile into oracle/_ref/libtrisolve.so (git-ignored; travels to the GPU box).
 */
#include <stdint.h>

int tri_forward(int64_t n, const int64_t* ptr, const int32_t* col, const double* val, const double* b,
                double* x) {
  for (int64_t i = 0; i < n; ++i) {
    double s = b[i], d = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
      const int64_t j = col[k];
      if (j < i) s -= val[k] * x[j];
      else if (j == i) d = val[k];
      else break;
    }
    if (d == 0.0) return -1;
    x[i] = s / d;
  }
  return 0;
}

int tri_backward(int64_t n, const int64_t* ptr, const int32_t* col, const double* val, const double* b,
                 double* x) {
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = b[i], d = 0.0;
    for (int64_t k = ptr[i + 1] - 1; k >= ptr[i]; --k) {
      const int64_t j = col[k];
      if (j > i) s -= val[k] * x[j];
      else if (j == i) d = val[k];
      else break;
    }
    if (d == 0.0) return -1;
    x[i] = s / d;
  }
  return 0;
}
