/*
 * hpdinv_oracle.h -- plain, slow, obviously-correct CPU oracle (fp64 / complex128).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1111_4144_b200/, include/hpdinv.h) never includes, links or calls it, and this
 * oracle shares no code, header, table or helper with the CUDA path.
 *
 * Every routine follows "Matrix Inversion Using Cholesky Decomposition"
 * (arxiv/paper_1111_4144, /root/reference/PAPER.md, cited as P:<line>) step by step, in the
 * paper's order and notation, with 0-based C indices (the paper is 1-based).
 *
 * Matrices are dense, row-major, n x n, `double complex` (C99).  Factors are upper
 * triangular (R = L*); entries strictly below the diagonal of R are set to 0.
 *
 * Counting: every routine takes an optional `oracle_counts *` (NULL = do not count).  One
 * complex multiply (including r*_ki r_ki, eq. 3) counts 1 in `cmul`; a division by a pivot
 * counts 1 in `cdiv`; a square root 1 in `csqrt`; a complex add/sub 1 in `cadd`
 * (Table 1, P:212-219 counts multiplies at complex-element granularity; reading R12).
 */
#ifndef HPDINV_ORACLE_H
#define HPDINV_ORACLE_H

#include <complex.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    long long cmul;   /* complex multiplies (Table 1 "operations")          */
    long long cdiv;   /* divisions by a pivot r_ii or d_i                   */
    long long cadd;   /* complex additions / subtractions                    */
    long long csqrt;  /* square roots (eq. 3 only; LDL has none)       */
} oracle_counts;

/* Counting conventions for the two existing methods (reading R10). */
enum {
    ORACLE_PAPER_CONVENTION = 0,   /* skip structurally-zero rows, full-length dot products */
    ORACLE_FULL_EXPLOITATION = 1   /* also truncate dot products at structural zeros        */
};

/* Cholesky A = R*R, eqs. (3)-(4).  Reads only a_ij with i <= j and Re(a_ii).
 * Returns info: 0 on success, else the first 1-based pivot i with !(t_i > 0), where
 * t_i = Re a_ii - sum_{k<i} r*_ki r_ki is the radicand of eq. (3) (reading R6).
 * On failure R is left partially written. */
int oracle_chol_upper(int n, const double complex *A, double complex *R, oracle_counts *c);

/* LDL A = R*DR, eqs. (10)-(11), R unit upper triangular, D = diag(d).
 * w_k = d_k r*_ki is cached per row so the cost equals Cholesky's.
 * Returns info: first 1-based i with !(d_i > 0), else 0. */
int oracle_ldl_upper(int n, const double complex *A, double complex *R, double *d,
                     oracle_counts *c);

/* Proposed method, Cholesky, eqs. (20)-(24): back-substitution R x_i = s_i with
 * S = diag(1/r_ii) (eq. 24), solving only x_kj, k <= j, using x_jm = conj(x_mj) where needed
 * (P:175-176), then the Hermitian mirror.  Writes the full X. */
void oracle_proposed_inv_chol(int n, const double complex *R, double complex *X, oracle_counts *c);

/* Proposed method, LDL, eqs. (25)-(29): unit R, S~ = diag(1/d_i) (eq. 29). */
void oracle_proposed_inv_ldl(int n, const double complex *R, const double *d, double complex *X,
                             oracle_counts *c);

/* Hermitian mirror: x_ji = conj(x_ij) for i < j; Im x_ii := 0. */
void oracle_mirror(int n, double complex *X);

/* Existing method A, equation solving, eq. (15): for every column i solve
 * R* b_i = e_i (eq. 6) then R x_i = b_i (eq. 7) for the upper half, then mirror. */
void oracle_eqsolve_inv(int n, const double complex *R, double complex *X, int convention,
                        oracle_counts *c);

/* Existing method B, triangular matrix operations, eqs. (16)-(19), P:115-133:
 * M = R^-1 via R m_i = e_i (eq. 18), X = M M* (eq. 19, upper half), then mirror. */
void oracle_trimat_inv(int n, const double complex *R, double complex *X, int convention,
                       oracle_counts *c);

/* Linear solve A x = y with Cholesky factor, eqs. (5)-(7), P:49-61 (one right-hand side). */
void oracle_solve_chol(int n, const double complex *R, const double complex *y, double complex *x,
                       oracle_counts *c);

/* Linear solve A x = y with LDL factors, eqs. (12)-(14). */
void oracle_solve_ldl(int n, const double complex *R, const double *d, const double complex *y,
                      double complex *x, oracle_counts *c);

/* Non-Hermitian extension: A = D D*, X = A^-1 (proposed method), D^-1 = D* X.
 * Returns the Cholesky info of A = DD*. */
int oracle_nonhermitian_inv(int n, const double complex *D, double complex *Dinv);

/* Batched driver over strided storage: element (i,j) of matrix b lives at
 * base[b*stride_mat + (i*n + j)*stride_elem].  method 0 = Cholesky + proposed (eqs. 3-4,
 * 20-24), 1 = LDL + proposed (eqs. 10-11, 25-29), 2 = Cholesky + equation solving (eq. 15),
 * 3 = Cholesky + triangular ops (eqs. 16-19).  Writes all n*n entries of X_b and info[b];
 * X_b is filled with NaN when info[b] != 0.  OpenMP across matrices only (nthreads <= 0:
 * library default).  Returns 0, or -1 on a bad argument. */
int oracle_inv_batched(int64_t batch, int n, const double complex *A, int64_t sA_mat,
                       int64_t sA_elem, double complex *X, int64_t sX_mat, int64_t sX_elem,
                       int32_t *info, int method, int nthreads);

/* Batched linear solve A_b x_b = y_b (method 0 Cholesky eqs. 5-7, 1 LDL eqs. 12-14).
 * y, x: batch x n, contiguous. */
int oracle_solve_batched(int64_t batch, int n, const double complex *A, int64_t sA_mat,
                         int64_t sA_elem, const double complex *y, double complex *x,
                         int32_t *info, int method, int nthreads);

/* Batched non-Hermitian inversion: contiguous batch x n x n D and Dinv;
 * info[b] = the Cholesky info of D_b D_b*. */
int oracle_nonherm_batched(int64_t batch, int n, const double complex *D, double complex *Dinv,
                           int32_t *info, int nthreads);

/* Number of OpenMP threads a parallel region would use (for the reported core count). */
int oracle_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
