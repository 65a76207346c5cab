/*
 * fxp_oracle.h -- fixed-point (Q-format) emulation of the inversion methods (§IV.C, P:206-208;
 * SURVEY §8(f) row f4).  TEST INFRASTRUCTURE ONLY (see hpdinv_oracle.h); arithmetic rules F1-F7
 * in fxp_oracle.c and DESIGN.md.
 *
 * A, X: n x n row-major, each complex entry an interleaved (re, im) pair of int64 raws of
 * Q(m, f) (value = raw * 2^-f).  Only the upper triangle and Re a_ii of A are read.
 * method: 0 = Cholesky + proposed inversion (eqs. 3-4, 20-24), 1 = equation solving (eq. 15),
 * 2 = triangular matrix operations (eqs. 16-19).  Returns the Cholesky info (0, or the first
 * 1-based pivot whose radicand is <= 0; X is zero then), or -1 for a bad argument; *nsat =
 * number of saturation events (F2).
 */
#ifndef FXP_ORACLE_H
#define FXP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int oracle_fxp_inv(int n, const int64_t *A, int64_t *X, int m, int f, int method, long long *nsat);

/* one operation for the pins: op 0 = F4 product a*b, 1 = F5 quotient a / bre (bre > 0),
 * 2 = F6 root of are (> 0); out = (re, im) raws; returns the saturation count */
int oracle_fxp_op(int op, int m, int f, int64_t are, int64_t aim, int64_t bre, int64_t bim, int64_t *out);

/* contiguous batch of matrices; info[b], nsat[b] per matrix; OpenMP across matrices only */
int oracle_fxp_inv_batched(int64_t batch, int n, const int64_t *A, int64_t *X, int32_t *info,
                           int64_t *nsat, int m, int f, int method, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
