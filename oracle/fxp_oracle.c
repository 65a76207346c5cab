/*
 * fxp_oracle.c -- fixed-point (Q-format) emulation of the three inversion methods, for the
 * paper's fixed-point accuracy study (§IV.C).
 *
 * TEST INFRASTRUCTURE ONLY (see hpdinv_oracle.h): shares no code with the CUDA path.
 *
 * The paper gives no word length, rounding or accumulation rule (Fig. 1 absent,
 * P:221); the arithmetic below is DESIGN.md's reading F1-F7 (after SPEC.md's QFormat /
 * quantize / fxp_mul):
 *   F1  Q(m, f): a value is raw * 2^-f, raw an integer in [-2^(m+f), 2^(m+f) - 1];
 *       1 <= m, 1 <= f, m + f <= 40 (products of two raws are exact in 128 bits).
 *   F2  every result is saturated to that range (saturation events are counted).
 *   F3  add / subtract / negate: exact, then F2.
 *   F4  complex multiply: the four real products exact (2f fractional bits), the real and
 *       imaginary sums exact, each rounded ONCE to f bits, round-half-to-even, then F2.
 *   F5  division by a positive real pivot p: round-half-even(a * 2^f / p), then F2.
 *   F6  square root of a positive real t: round-to-nearest(sqrt(t * 2^f)) (exact integer
 *       square root; no ties exist), then F2.
 *   F7  dot products accumulate term by term in the paper's index order with F3 after every
 *       F4-rounded product (no wide accumulator).
 * The methods follow the fp64 oracle's loops exactly (hpdinv_oracle.c): Cholesky eqs. (3)-(4);
 * proposed inversion eqs. (20)-(24); equation solving eq. (15); triangular ops eqs. (16)-(19).
 * Storage: complex raws as interleaved (re, im) int64 pairs, row-major n x n.
 */
#include "fxp_oracle.h"

#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __int128 i128;
typedef unsigned __int128 u128;
typedef struct { int64_t re, im; } fxc;
typedef struct { int m, f; int64_t lo, hi; long long nsat; } fxq;

static int64_t sat(fxq *q, i128 v)
{
    if (v > (i128)q->hi) { q->nsat++; return q->hi; }
    if (v < (i128)q->lo) { q->nsat++; return q->lo; }
    return (int64_t)v;
}

/* floor(v / 2^f) and the remainder, then round half to even */
static i128 rne_shift(i128 v, int f)
{
    i128 d = (i128)1 << f;
    i128 q = v / d, r = v % d;
    if (r < 0) { q -= 1; r += d; }                   /* floor division */
    i128 twice = 2 * r;
    if (twice > d || (twice == d && (q & 1))) q += 1;
    return q;
}

/* round half to even of num / den, den > 0 */
static i128 rne_div(i128 num, i128 den)
{
    i128 q = num / den, r = num % den;
    if (r < 0) { q -= 1; r += den; }
    i128 twice = 2 * r;
    if (twice > den || (twice == den && (q & 1))) q += 1;
    return q;
}

static fxc fadd(fxq *q, fxc a, fxc b) { fxc z = { sat(q, (i128)a.re + b.re), sat(q, (i128)a.im + b.im) }; return z; }
static fxc fsub(fxq *q, fxc a, fxc b) { fxc z = { sat(q, (i128)a.re - b.re), sat(q, (i128)a.im - b.im) }; return z; }

/* F4: a * b with a and/or b conjugated as asked */
static fxc fmul(fxq *q, fxc a, int conja, fxc b, int conjb)
{
    i128 ai = conja ? -(i128)a.im : (i128)a.im;
    i128 bi = conjb ? -(i128)b.im : (i128)b.im;
    i128 re = (i128)a.re * b.re - ai * bi;
    i128 im = (i128)a.re * bi + ai * b.re;
    fxc z = { sat(q, rne_shift(re, q->f)), sat(q, rne_shift(im, q->f)) };
    return z;
}

/* F5: a / p, p > 0 real */
static fxc fdiv(fxq *q, fxc a, int64_t p)
{
    fxc z = { sat(q, rne_div((i128)a.re << q->f, p)), sat(q, rne_div((i128)a.im << q->f, p)) };
    return z;
}

/* F6: round(sqrt(t * 2^f)), t > 0 */
static int64_t fsqrt(fxq *q, int64_t t)
{
    u128 x = (u128)t << q->f;
    /* floor sqrt by bisection over [0, 2^64) (plain, obviously correct) */
    u128 lo = 0, hi = (u128)1 << 64;
    while (hi - lo > 1) {
        u128 mid = (lo + hi) / 2;
        if (mid * mid <= x) lo = mid; else hi = mid;
    }
    if (x - lo * lo > lo) lo += 1;                    /* x > r^2 + r  <=>  sqrt(x) > r + 1/2 */
    return sat(q, (i128)lo);
}

#define IX(i, j) ((size_t)(i) * (size_t)n + (size_t)(j))

/* x~_mj = x_mj (m <= j) or conj(x_jm) (m > j): the stored entry and whether to
   conjugate it (the conjugation is applied exactly inside the F4 product) */
#define XT(X, m, j) ((m) <= (j) ? (X)[IX(m, j)] : (X)[IX(j, m)])
#define XC(m, j) ((m) > (j))

/* Cholesky, eqs. (3)-(4): returns info (first 1-based pivot with t <= 0) */
static int fx_chol(fxq *q, int n, const fxc *A, fxc *R)
{
    memset(R, 0, sizeof(fxc) * (size_t)n * n);
    for (int i = 0; i < n; i++) {
        fxc s = { 0, 0 };
        for (int k = 0; k < i; k++) s = fadd(q, s, fmul(q, R[IX(k, i)], 1, R[IX(k, i)], 0));
        int64_t t = sat(q, (i128)A[IX(i, i)].re - s.re);
        if (!(t > 0)) return i + 1;
        int64_t rii = fsqrt(q, t);
        if (!(rii > 0)) return i + 1;
        R[IX(i, i)].re = rii;
        R[IX(i, i)].im = 0;
        for (int j = i + 1; j < n; j++) {
            fxc sj = { 0, 0 };
            for (int k = 0; k < i; k++) sj = fadd(q, sj, fmul(q, R[IX(k, i)], 1, R[IX(k, j)], 0));
            R[IX(i, j)] = fdiv(q, fsub(q, A[IX(i, j)], sj), rii);
        }
    }
    return 0;
}

static void fx_mirror(fxq *q, int n, fxc *X)
{
    for (int i = 0; i < n; i++) {
        X[IX(i, i)].im = 0;
        for (int j = i + 1; j < n; j++) {
            X[IX(j, i)].re = X[IX(i, j)].re;
            X[IX(j, i)].im = sat(q, -(i128)X[IX(i, j)].im);
        }
    }
}

/* proposed inversion, eqs. (20)-(24), in the fp64 oracle's order */
static void fx_proposed(fxq *q, int n, const fxc *R, fxc *X)
{
    const fxc zero = { 0, 0 };
    const fxc one = { (int64_t)1 << q->f, 0 };
    memset(X, 0, sizeof(fxc) * (size_t)n * n);
    for (int k = n - 1; k >= 0; k--) {
        int64_t rkk = R[IX(k, k)].re;
        for (int j = k + 1; j < n; j++) {
            fxc s = zero;
            for (int m = k + 1; m < n; m++) s = fadd(q, s, fmul(q, R[IX(k, m)], 0, XT(X, m, j), XC(m, j)));
            X[IX(k, j)] = fdiv(q, fsub(q, zero, s), rkk);
        }
        fxc s = zero;
        for (int m = k + 1; m < n; m++) s = fadd(q, s, fmul(q, R[IX(k, m)], 0, XT(X, m, k), XC(m, k)));
        fxc skk = fdiv(q, one, rkk);                   /* eq. (24) */
        fxc d = { sat(q, (i128)skk.re - s.re), 0 };
        X[IX(k, k)] = fdiv(q, d, rkk);
        X[IX(k, k)].im = 0;
    }
    fx_mirror(q, n, X);
}

/* equation solving, eq. (15): columns N..1, forward R* b = e_i (rows >= i), back R x_i = b */
static void fx_eqsolve(fxq *q, int n, const fxc *R, fxc *X)
{
    const fxc zero = { 0, 0 };
    fxc *b = (fxc *)calloc((size_t)n + 1, sizeof(fxc));
    memset(X, 0, sizeof(fxc) * (size_t)n * n);
    for (int i = n - 1; i >= 0; i--) {
        for (int k = 0; k < n; k++) b[k] = zero;
        for (int k = i; k < n; k++) {
            fxc s = zero;
            for (int p = i; p < k; p++) s = fadd(q, s, fmul(q, R[IX(p, k)], 1, b[p], 0));
            fxc e = { k == i ? ((int64_t)1 << q->f) : 0, 0 };
            b[k] = fdiv(q, fsub(q, e, s), R[IX(k, k)].re);
        }
        for (int k = i; k >= 0; k--) {
            fxc s = zero;
            for (int m = k + 1; m < n; m++) s = fadd(q, s, fmul(q, R[IX(k, m)], 0, XT(X, m, i), XC(m, i)));
            X[IX(k, i)] = fdiv(q, fsub(q, b[k], s), R[IX(k, k)].re);
        }
    }
    free(b);
    fx_mirror(q, n, X);
}

/* triangular matrix operations, eqs. (16)-(19): M = R^-1 (rows k <= i), X = M M* upper */
static void fx_trimat(fxq *q, int n, const fxc *R, fxc *X)
{
    const fxc zero = { 0, 0 };
    fxc *M = (fxc *)calloc((size_t)n * n + 1, sizeof(fxc));
    memset(X, 0, sizeof(fxc) * (size_t)n * n);
    for (int i = 0; i < n; i++)
        for (int k = i; k >= 0; k--) {
            fxc s = zero;
            for (int m = k + 1; m <= i; m++) s = fadd(q, s, fmul(q, R[IX(k, m)], 0, M[IX(m, i)], 0));
            fxc e = { k == i ? ((int64_t)1 << q->f) : 0, 0 };
            M[IX(k, i)] = fdiv(q, fsub(q, e, s), R[IX(k, k)].re);
        }
    for (int i = 0; i < n; i++)
        for (int j = i; j < n; j++) {
            fxc s = zero;
            for (int p = j; p < n; p++) s = fadd(q, s, fmul(q, M[IX(i, p)], 0, M[IX(j, p)], 1));
            X[IX(i, j)] = s;
        }
    free(M);
    fx_mirror(q, n, X);
}

/* single F4 product / F5 quotient / F6 root for the pins (out: re, im raws; returns nsat) */
int oracle_fxp_op(int op, int m, int f, int64_t are, int64_t aim, int64_t bre, int64_t bim, int64_t *out)
{
    fxq q = { m, f, -((int64_t)1 << (m + f)), ((int64_t)1 << (m + f)) - 1, 0 };
    fxc a = { are, aim }, b = { bre, bim }, z = { 0, 0 };
    if (op == 0) z = fmul(&q, a, 0, b, 0);
    else if (op == 1) z = fdiv(&q, a, bre);
    else z.re = fsqrt(&q, are);
    out[0] = z.re;
    out[1] = z.im;
    return (int)q.nsat;
}

int oracle_fxp_inv(int n, const int64_t *A, int64_t *X, int m, int f, int method, long long *nsat)
{
    if (n < 1 || m < 1 || f < 1 || m + f > 40 || method < 0 || method > 2) return -1;
    fxq q = { m, f, -((int64_t)1 << (m + f)), ((int64_t)1 << (m + f)) - 1, 0 };
    size_t nn = (size_t)n * n;
    fxc *a = (fxc *)malloc(sizeof(fxc) * nn), *r = (fxc *)malloc(sizeof(fxc) * nn),
        *x = (fxc *)malloc(sizeof(fxc) * nn);
    for (size_t e = 0; e < nn; e++) { a[e].re = A[2 * e]; a[e].im = A[2 * e + 1]; }
    int info = fx_chol(&q, n, a, r);
    if (info == 0) {
        if (method == 0) fx_proposed(&q, n, r, x);
        else if (method == 1) fx_eqsolve(&q, n, r, x);
        else fx_trimat(&q, n, r, x);
        for (size_t e = 0; e < nn; e++) { X[2 * e] = x[e].re; X[2 * e + 1] = x[e].im; }
    } else {
        for (size_t e = 0; e < 2 * nn; e++) X[e] = 0;
    }
    if (nsat) *nsat = q.nsat;
    free(a); free(r); free(x);
    return info;
}

int oracle_fxp_inv_batched(int64_t batch, int n, const int64_t *A, int64_t *X, int32_t *info,
                           int64_t *nsat, int m, int f, int method, int nthreads)
{
    if (batch < 0 || n < 1 || m < 1 || f < 1 || m + f > 40 || method < 0 || method > 2) return -1;
    size_t stride = 2 * (size_t)n * n;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int64_t b = 0; b < batch; b++) {
        long long ns = 0;
        info[b] = oracle_fxp_inv(n, A + b * stride, X + b * stride, m, f, method, &ns);
        nsat[b] = ns;
    }
    return 0;
}
