/*
 * hpdinv_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY (see hpdinv_oracle.h).  Nothing here is blocked, fused or
 * reordered beyond what the paper's equations state; loops run in the paper's index
 * order.  0-based indices in code; comments quote the paper's 1-based notation.
 * Citations: P:<line> = /root/reference/PAPER.md line.
 *
 * Build: gcc -O2 -std=c11 -fopenmp -ffp-contract=off -fPIC -shared (see oracle/__init__.py).
 */
#include "hpdinv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define IDX(i, j) ((size_t)(i) * (size_t)n + (size_t)(j))
#define CMUL(c) do { if (c) (c)->cmul++; } while (0)
#define CDIV(c) do { if (c) (c)->cdiv++; } while (0)
#define CADD(c) do { if (c) (c)->cadd++; } while (0)
#define CSQRT(c) do { if (c) (c)->csqrt++; } while (0)

/* ---------------------------------------------------------------- Cholesky, eqs. (3)-(4) */
int oracle_chol_upper(int n, const double complex *A, double complex *R, oracle_counts *c)
{
    for (int i = 0; i < n * n; i++) R[i] = 0.0;
    for (int i = 0; i < n; i++) {
        /* eq. (3): r_ii = sqrt(a_ii - sum_{k=1}^{i-1} r*_ki r_ki) */
        double complex s = 0.0;
        for (int k = 0; k < i; k++) {
            s += conj(R[IDX(k, i)]) * R[IDX(k, i)];
            CMUL(c); CADD(c);
        }
        double t = creal(A[IDX(i, i)]) - creal(s);   /* a_ii is real for Hermitian A */
        CADD(c);
        if (!(t > 0.0)) return i + 1;                  /* not positive definite at pivot i */
        double rii = sqrt(t);
        CSQRT(c);
        R[IDX(i, i)] = rii;
        /* eq. (4): r_ij = (a_ij - sum_{k=1}^{i-1} r*_ki r_kj) / r_ii,  i < j */
        for (int j = i + 1; j < n; j++) {
            double complex sj = 0.0;
            for (int k = 0; k < i; k++) {
                sj += conj(R[IDX(k, i)]) * R[IDX(k, j)];
                CMUL(c); CADD(c);
            }
            R[IDX(i, j)] = (A[IDX(i, j)] - sj) / rii;
            CADD(c); CDIV(c);
        }
    }
    return 0;
}

/* --------------------------------------------------------------------- LDL, eqs. (10)-(11) */
int oracle_ldl_upper(int n, const double complex *A, double complex *R, double *d,
                     oracle_counts *c)
{
    double complex *w = (double complex *)malloc(sizeof(double complex) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n * n; i++) R[i] = 0.0;
    for (int i = 0; i < n; i++) d[i] = 0.0;
    int info = 0;
    for (int i = 0; i < n; i++) {
        /* "efficiently implemented": w_k = r*_ki d_k is formed once per row i
           (a real scaling, not a complex multiply) and reused by eqs. (10) and (11). */
        for (int k = 0; k < i; k++) w[k] = conj(R[IDX(k, i)]) * d[k];
        /* eq. (10): d_i = a_ii - sum_{k=1}^{i-1} r*_ki r_ki d_k */
        double complex s = 0.0;
        for (int k = 0; k < i; k++) {
            s += w[k] * R[IDX(k, i)];
            CMUL(c); CADD(c);
        }
        double di = creal(A[IDX(i, i)]) - creal(s);
        CADD(c);
        d[i] = di;
        if (!(di > 0.0)) { info = i + 1; break; }    /* flags non-PD (reading R6) */
        R[IDX(i, i)] = 1.0;
        /* eq. (11): r_ij = (a_ij - sum_{k=1}^{i-1} r*_ki r_kj d_k) / d_i,  i < j */
        for (int j = i + 1; j < n; j++) {
            double complex sj = 0.0;
            for (int k = 0; k < i; k++) {
                sj += w[k] * R[IDX(k, j)];
                CMUL(c); CADD(c);
            }
            R[IDX(i, j)] = (A[IDX(i, j)] - sj) / di;
            CADD(c); CDIV(c);
        }
    }
    free(w);
    return info;
}

/* ------------------------------------------------------------------- mirror */
void oracle_mirror(int n, double complex *X)
{
    for (int i = 0; i < n; i++) {
        X[IDX(i, i)] = creal(X[IDX(i, i)]);
        for (int j = i + 1; j < n; j++) X[IDX(j, i)] = conj(X[IDX(i, j)]);
    }
}

/* x~_mj: the (m,j) entry of X taken from the upper half, x_mj = conj(x_jm) when m > j
   ("x_ji = x*_ij where needed"). */
static double complex xt(int n, const double complex *X, int m, int j)
{
    return (m <= j) ? X[IDX(m, j)] : conj(X[IDX(j, m)]);
}

/* ----------------------------------------- proposed method, Cholesky, eqs. (20)-(24) */
void oracle_proposed_inv_chol(int n, const double complex *R, double complex *X, oracle_counts *c)
{
    for (int i = 0; i < n * n; i++) X[i] = 0.0;
    /* R X = B (eq. 23) with the upper part of B known without solving eq. (22):
       s_ij = 1/l_ii = 1/r_ii if i = j, 0 otherwise (eq. 24, reading R1).  Back-substitution
       R x_j = s_j, rows k = N..1; only x_kj with k <= j are solved (reading R2). */
    for (int k = n - 1; k >= 0; k--) {
        double rkk = creal(R[IDX(k, k)]);
        /* off-diagonal entries of row k: r_kk x_kj + sum_{m>k} r_km x_mj = s_kj = 0 */
        for (int j = k + 1; j < n; j++) {
            double complex s = 0.0;
            for (int m = k + 1; m < n; m++) {
                s += R[IDX(k, m)] * xt(n, X, m, j);
                CMUL(c); CADD(c);
            }
            X[IDX(k, j)] = (0.0 - s) / rkk;
            CADD(c); CDIV(c);
        }
        /* diagonal: r_kk x_kk + sum_{m>k} r_km x_mk = s_kk = 1/r_kk, with x_mk = conj(x_km);
           x_kk is real (X Hermitian), formed from the real part (reading R4). */
        double complex s = 0.0;
        for (int m = k + 1; m < n; m++) {
            s += R[IDX(k, m)] * xt(n, X, m, k);
            CMUL(c); CADD(c);
        }
        double skk = 1.0 / rkk;                         /* eq. (24) */
        CDIV(c);
        X[IDX(k, k)] = (skk - creal(s)) / rkk;
        CADD(c); CDIV(c);
    }
    oracle_mirror(n, X);
}

/* ------------------------------------------------------ proposed method, LDL, eqs. (25)-(29) */
void oracle_proposed_inv_ldl(int n, const double complex *R, const double *d, double complex *X,
                             oracle_counts *c)
{
    for (int i = 0; i < n * n; i++) X[i] = 0.0;
    /* R X = B~ (eq. 28), R unit upper; upper part of B~ is S~ = diag(1/d_i) (eq. 29). */
    for (int k = n - 1; k >= 0; k--) {
        for (int j = k + 1; j < n; j++) {
            double complex s = 0.0;
            for (int m = k + 1; m < n; m++) {
                s += R[IDX(k, m)] * xt(n, X, m, j);
                CMUL(c); CADD(c);
            }
            X[IDX(k, j)] = 0.0 - s;                      /* r_kk = 1 */
            CADD(c);
        }
        double complex s = 0.0;
        for (int m = k + 1; m < n; m++) {
            s += R[IDX(k, m)] * xt(n, X, m, k);
            CMUL(c); CADD(c);
        }
        double skk = 1.0 / d[k];                         /* eq. (29) */
        CDIV(c);
        X[IDX(k, k)] = skk - creal(s);
        CADD(c);
    }
    oracle_mirror(n, X);
}

/* ----------------------------------------------- existing method A: equation solving, eq. (15) */
void oracle_eqsolve_inv(int n, const double complex *R, double complex *X, int convention,
                        oracle_counts *c)
{
    double complex *b = (double complex *)malloc(sizeof(double complex) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n * n; i++) X[i] = 0.0;
    /* Columns are solved i = N..1 so that the lower entries x_mi = conj(x_im), m > i, needed
       by the back-substitution of column i are already known. */
    for (int i = n - 1; i >= 0; i--) {
        /* eq. (6): R* b = e_i, forward substitution; rows k < i are structurally zero. */
        for (int k = 0; k < n; k++) b[k] = 0.0;
        for (int k = i; k < n; k++) {
            int p0 = (convention == ORACLE_FULL_EXPLOITATION) ? i : 0;
            double complex s = 0.0;
            for (int p = p0; p < k; p++) {
                s += conj(R[IDX(p, k)]) * b[p];
                CMUL(c); CADD(c);
            }
            double complex e = (k == i) ? 1.0 : 0.0;
            b[k] = (e - s) / creal(R[IDX(k, k)]);
            CADD(c); CDIV(c);
        }
        /* eq. (7): R x_i = b, backward substitution for the upper half, rows k = i..1. */
        for (int k = i; k >= 0; k--) {
            double complex s = 0.0;
            for (int m = k + 1; m < n; m++) {
                s += R[IDX(k, m)] * xt(n, X, m, i);
                CMUL(c); CADD(c);
            }
            X[IDX(k, i)] = (b[k] - s) / creal(R[IDX(k, k)]);
            CADD(c); CDIV(c);
        }
    }
    free(b);
    oracle_mirror(n, X);
}

/* ------------------------------------- existing method B: triangular matrix ops, eqs. (16)-(19) */
void oracle_trimat_inv(int n, const double complex *R, double complex *X, int convention,
                       oracle_counts *c)
{
    double complex *M = (double complex *)calloc((size_t)n * (size_t)n + 1, sizeof(double complex));
    for (int i = 0; i < n * n; i++) X[i] = 0.0;
    /* eq. (18): R m_i = e_i; M = R^-1 is upper triangular, so only rows k <= i are solved. */
    for (int i = 0; i < n; i++) {
        for (int k = i; k >= 0; k--) {
            int m1 = (convention == ORACLE_FULL_EXPLOITATION) ? i + 1 : n;
            double complex s = 0.0;
            for (int m = k + 1; m < m1; m++) {
                s += R[IDX(k, m)] * M[IDX(m, i)];
                CMUL(c); CADD(c);
            }
            double complex e = (k == i) ? 1.0 : 0.0;
            M[IDX(k, i)] = (e - s) / creal(R[IDX(k, k)]);
            CADD(c); CDIV(c);
        }
    }
    /* eq. (19): X = M M*, upper half: x_ij = sum_p m_ip conj(m_jp), nonzero terms p >= j. */
    for (int i = 0; i < n; i++) {
        for (int j = i; j < n; j++) {
            double complex s = 0.0;
            for (int p = j; p < n; p++) {
                s += M[IDX(i, p)] * conj(M[IDX(j, p)]);
                CMUL(c); CADD(c);
            }
            X[IDX(i, j)] = s;
        }
    }
    free(M);
    oracle_mirror(n, X);
}

/* ------------------------------------------------------ linear solves, eqs. (5)-(7), (12)-(14) */
void oracle_solve_chol(int n, const double complex *R, const double complex *y, double complex *x,
                       oracle_counts *c)
{
    double complex *b = (double complex *)malloc(sizeof(double complex) * (size_t)(n > 0 ? n : 1));
    /* eq. (6): R* b = y (forward substitution; the paper calls it backward, reading R8) */
    for (int k = 0; k < n; k++) {
        double complex s = 0.0;
        for (int p = 0; p < k; p++) { s += conj(R[IDX(p, k)]) * b[p]; CMUL(c); CADD(c); }
        b[k] = (y[k] - s) / creal(R[IDX(k, k)]);
        CADD(c); CDIV(c);
    }
    /* eq. (7): R x = b (backward substitution) */
    for (int k = n - 1; k >= 0; k--) {
        double complex s = 0.0;
        for (int m = k + 1; m < n; m++) { s += R[IDX(k, m)] * x[m]; CMUL(c); CADD(c); }
        x[k] = (b[k] - s) / creal(R[IDX(k, k)]);
        CADD(c); CDIV(c);
    }
    free(b);
}

void oracle_solve_ldl(int n, const double complex *R, const double *d, const double complex *y,
                      double complex *x, oracle_counts *c)
{
    double complex *b = (double complex *)malloc(sizeof(double complex) * (size_t)(n > 0 ? n : 1));
    /* eq. (13): R* D b = y; row k: sum_{p<=k} conj(r_pk) d_p b_p = y_k, r_kk = 1 */
    for (int k = 0; k < n; k++) {
        double complex s = 0.0;
        for (int p = 0; p < k; p++) { s += conj(R[IDX(p, k)]) * (d[p] * b[p]); CMUL(c); CADD(c); }
        b[k] = (y[k] - s) / d[k];
        CADD(c); CDIV(c);
    }
    /* eq. (14): R x = b, unit upper */
    for (int k = n - 1; k >= 0; k--) {
        double complex s = 0.0;
        for (int m = k + 1; m < n; m++) { s += R[IDX(k, m)] * x[m]; CMUL(c); CADD(c); }
        x[k] = b[k] - s;
        CADD(c);
    }
    free(b);
}

/* ---------------------------------------------------- non-Hermitian extension */
int oracle_nonhermitian_inv(int n, const double complex *D, double complex *Dinv)
{
    size_t nn = (size_t)n * (size_t)n;
    double complex *A = (double complex *)calloc(nn + 1, sizeof(double complex));
    double complex *R = (double complex *)calloc(nn + 1, sizeof(double complex));
    double complex *X = (double complex *)calloc(nn + 1, sizeof(double complex));
    /* A = D D*: a_ij = sum_p d_ip conj(d_jp) */
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) {
            double complex s = 0.0;
            for (int p = 0; p < n; p++) s += D[IDX(i, p)] * conj(D[IDX(j, p)]);
            A[IDX(i, j)] = s;
        }
    int info = oracle_chol_upper(n, A, R, NULL);
    if (info == 0) {
        oracle_proposed_inv_chol(n, R, X, NULL);
        /* D^-1 = D* A^-1: (D^-1)_ij = sum_p conj(d_pi) x_pj */
        for (int i = 0; i < n; i++)
            for (int j = 0; j < n; j++) {
                double complex s = 0.0;
                for (int p = 0; p < n; p++) s += conj(D[IDX(p, i)]) * X[IDX(p, j)];
                Dinv[IDX(i, j)] = s;
            }
    } else {
        for (size_t i = 0; i < nn; i++) Dinv[i] = NAN;
    }
    free(A); free(R); free(X);
    return info;
}

/* -------------------------------------------------------------------------- batched drivers */
static void load_upper(int n, const double complex *base, int64_t sm, int64_t se, int64_t b,
                       double complex *A)
{
    /* Only a_ij with i <= j are referenced by eqs. (3)-(4) and (10)-(11) (reading R5). */
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) {
            if (j < i) { A[IDX(i, j)] = 0.0; continue; }
            double complex v = base[b * sm + (int64_t)(i * n + j) * se];
            A[IDX(i, j)] = (i == j) ? creal(v) : v;
        }
}

int oracle_inv_batched(int64_t batch, int n, const double complex *A, int64_t sA_mat,
                       int64_t sA_elem, double complex *X, int64_t sX_mat, int64_t sX_elem,
                       int32_t *info, int method, int nthreads)
{
    if (batch < 0 || n < 1 || method < 0 || method > 3) return -1;
    if (batch == 0) return 0;
    if (!A || !X || !info) return -1;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
    {
        size_t nn = (size_t)n * (size_t)n;
        double complex *a = (double complex *)malloc(sizeof(double complex) * nn);
        double complex *r = (double complex *)malloc(sizeof(double complex) * nn);
        double complex *x = (double complex *)malloc(sizeof(double complex) * nn);
        double *d = (double *)malloc(sizeof(double) * (size_t)n);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t b = 0; b < batch; b++) {
            load_upper(n, A, sA_mat, sA_elem, b, a);
            int inf;
            if (method == 1) {
                inf = oracle_ldl_upper(n, a, r, d, NULL);
                if (inf == 0) oracle_proposed_inv_ldl(n, r, d, x, NULL);
            } else {
                inf = oracle_chol_upper(n, a, r, NULL);
                if (inf == 0) {
                    if (method == 0) oracle_proposed_inv_chol(n, r, x, NULL);
                    else if (method == 2) oracle_eqsolve_inv(n, r, x, ORACLE_PAPER_CONVENTION, NULL);
                    else oracle_trimat_inv(n, r, x, ORACLE_PAPER_CONVENTION, NULL);
                }
            }
            if (inf != 0)
                for (size_t e = 0; e < nn; e++) x[e] = NAN;
            for (int i = 0; i < n; i++)
                for (int j = 0; j < n; j++)
                    X[b * sX_mat + (int64_t)(i * n + j) * sX_elem] = x[IDX(i, j)];
            info[b] = inf;
        }
        free(a); free(r); free(x); free(d);
    }
    return 0;
}

int oracle_solve_batched(int64_t batch, int n, const double complex *A, int64_t sA_mat,
                         int64_t sA_elem, const double complex *y, double complex *x,
                         int32_t *info, int method, int nthreads)
{
    if (batch < 0 || n < 1 || method < 0 || method > 1) return -1;
    if (batch == 0) return 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
    {
        size_t nn = (size_t)n * (size_t)n;
        double complex *a = (double complex *)malloc(sizeof(double complex) * nn);
        double complex *r = (double complex *)malloc(sizeof(double complex) * nn);
        double *d = (double *)malloc(sizeof(double) * (size_t)n);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t b = 0; b < batch; b++) {
            load_upper(n, A, sA_mat, sA_elem, b, a);
            int inf = (method == 1) ? oracle_ldl_upper(n, a, r, d, NULL)
                                    : oracle_chol_upper(n, a, r, NULL);
            if (inf == 0) {
                if (method == 1) oracle_solve_ldl(n, r, d, y + b * n, x + b * n, NULL);
                else oracle_solve_chol(n, r, y + b * n, x + b * n, NULL);
            } else {
                for (int k = 0; k < n; k++) x[b * n + k] = NAN;
            }
            info[b] = inf;
        }
        free(a); free(r); free(d);
    }
    return 0;
}

/* Batched non-Hermitian inversion, one oracle_nonhermitian_inv per matrix.
 * D: contiguous batch x n x n; Dinv likewise; OpenMP across matrices only. */
int oracle_nonherm_batched(int64_t batch, int n, const double complex *D, double complex *Dinv,
                           int32_t *info, int nthreads)
{
    if (batch < 0 || n < 1) return -1;
    if (batch == 0) return 0;
    size_t nn = (size_t)n * (size_t)n;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int64_t b = 0; b < batch; b++)
        info[b] = oracle_nonhermitian_inv(n, D + (size_t)b * nn, Dinv + (size_t)b * nn);
    return 0;
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
