// k_fxp.cu -- fixed-point (Q-format) emulation of the three inversion methods on the GPU, for
// the paper's fixed-point accuracy study (§IV.C, Fig. 1).
//
// One matrix (one trial) per thread; the matrix, its factor and X live in the thread's local
// memory (the emulation is integer-ALU bound, not a dense contraction).  The arithmetic is
// DESIGN.md's reading F1-F7 -- the paper fixes none of it:
//   F1 Q(m, f): value = raw * 2^-f, raw in [-2^(m+f), 2^(m+f) - 1], 1 <= m, f; m + f <= 40;
//   F2 every result saturates to that range (events counted);
//   F3 add / subtract exact then F2;
//   F4 complex multiply: exact 128-bit products and sums, ONE round-half-to-even to f bits per
//      component, then F2;
//   F5 division by a positive real pivot: round-half-to-even(a 2^f / p), then F2;
//   F6 square root: round-to-nearest(sqrt(t 2^f)) from an exact integer square root;
//   F7 dot products accumulate term by term (index order of the paper's sums), F3 after every
//      F4 product.
// Methods (each after the Cholesky factor, eqs. 3-4): 0 proposed (eqs. 20-24), 1 equation
// solving (eq. 15), 2 triangular matrix operations (eqs. 16-19); loop orders are those of
// DESIGN.md §6 (f4), so the results are bit-exact against the fixed-point oracle.
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hpdinv.h"
#include "dispatch.h"

namespace hpdinv {
namespace fxp {

using i128 = __int128;
using u128 = unsigned __int128;

struct Fx { int64_t re, im; };
struct Q {
    int f;
    int64_t lo, hi;
    int64_t nsat;
    __device__ int64_t sat(i128 v) {
        if (v > i128(hi)) { nsat++; return hi; }
        if (v < i128(lo)) { nsat++; return lo; }
        return int64_t(v);
    }
};

// round half to even of v / 2^f (arithmetic shift = floor, remainder in [0, 2^f))
__device__ __forceinline__ i128 rshift_rne(i128 v, int f) {
    const i128 q = v >> f;
    const i128 r = v - (q << f);
    const i128 half = i128(1) << (f - 1);
    return (r > half || (r == half && (q & 1))) ? q + 1 : q;
}

// round half to even of num / den, den > 0
__device__ __forceinline__ i128 div_rne(i128 num, int64_t den) {
    i128 q = num / den;
    i128 r = num - q * den;                              // truncated toward zero
    if (r < 0) { q -= 1; r += den; }                     // -> floor
    const i128 twice = 2 * r;
    return (twice > den || (twice == den && (q & 1))) ? q + 1 : q;
}

__device__ __forceinline__ Fx add(Q& q, Fx a, Fx b) { return Fx{q.sat(i128(a.re) + b.re), q.sat(i128(a.im) + b.im)}; }
__device__ __forceinline__ Fx sub(Q& q, Fx a, Fx b) { return Fx{q.sat(i128(a.re) - b.re), q.sat(i128(a.im) - b.im)}; }

// F4: (conj(a) if ca) * (conj(b) if cb)
__device__ __forceinline__ Fx mul(Q& q, Fx a, bool ca, Fx b, bool cb) {
    const i128 ai = ca ? -i128(a.im) : i128(a.im);
    const i128 bi = cb ? -i128(b.im) : i128(b.im);
    const i128 re = i128(a.re) * b.re - ai * bi;
    const i128 im = i128(a.re) * bi + ai * b.re;
    return Fx{q.sat(rshift_rne(re, q.f)), q.sat(rshift_rne(im, q.f))};
}

__device__ __forceinline__ Fx divp(Q& q, Fx a, int64_t p) {
    return Fx{q.sat(div_rne(i128(a.re) << q.f, p)), q.sat(div_rne(i128(a.im) << q.f, p))};
}

// F6: nearest integer to sqrt(t 2^f); floor root from a double estimate, corrected exactly
__device__ __forceinline__ int64_t sqrtq(Q& q, int64_t t) {
    const u128 x = u128(t) << q.f;
    uint64_t r = uint64_t(sqrt(double(x)));
    while (u128(r) * r > x) r--;
    while (u128(r + 1) * (r + 1) <= x) r++;
    if (x - u128(r) * r > u128(r)) r++;
    return q.sat(i128(r));
}

template <int N>
__device__ int chol(Q& q, const Fx* A, Fx* R) {
    for (int e = 0; e < N * N; e++) R[e] = Fx{0, 0};
    for (int i = 0; i < N; i++) {
        Fx s{0, 0};
        for (int k = 0; k < i; k++) s = add(q, s, mul(q, R[k * N + i], true, R[k * N + i], false));
        const int64_t t = q.sat(i128(A[i * N + i].re) - s.re);
        if (!(t > 0)) return i + 1;
        const int64_t rii = sqrtq(q, t);
        if (!(rii > 0)) return i + 1;
        R[i * N + i] = Fx{rii, 0};
        for (int j = i + 1; j < N; j++) {
            Fx sj{0, 0};
            for (int k = 0; k < i; k++) sj = add(q, sj, mul(q, R[k * N + i], true, R[k * N + j], false));
            R[i * N + j] = divp(q, sub(q, A[i * N + j], sj), rii);
        }
    }
    return 0;
}

template <int N>
__device__ void mirror(Q& q, Fx* X) {
    for (int i = 0; i < N; i++) {
        X[i * N + i].im = 0;
        for (int j = i + 1; j < N; j++) X[j * N + i] = Fx{X[i * N + j].re, q.sat(-i128(X[i * N + j].im))};
    }
}

// x~_mj of the upper-stored X: (entry, conjugate?)
#define FXP_XT(X, m, j) ((m) <= (j) ? (X)[(m) * N + (j)] : (X)[(j) * N + (m)])

template <int N>
__device__ void proposed(Q& q, const Fx* R, Fx* X) {
    const Fx zero{0, 0}, one{int64_t(1) << q.f, 0};
    for (int e = 0; e < N * N; e++) X[e] = zero;
    for (int k = N - 1; k >= 0; k--) {
        const int64_t rkk = R[k * N + k].re;
        for (int j = k + 1; j < N; j++) {
            Fx s = zero;
            for (int m = k + 1; m < N; m++) s = add(q, s, mul(q, R[k * N + m], false, FXP_XT(X, m, j), m > j));
            X[k * N + j] = divp(q, sub(q, zero, s), rkk);
        }
        Fx s = zero;
        for (int m = k + 1; m < N; m++) s = add(q, s, mul(q, R[k * N + m], false, FXP_XT(X, m, k), m > k));
        const Fx skk = divp(q, one, rkk);                // eq. (24)
        X[k * N + k] = divp(q, Fx{q.sat(i128(skk.re) - s.re), 0}, rkk);
        X[k * N + k].im = 0;
    }
    mirror<N>(q, X);
}

template <int N>
__device__ void eqsolve(Q& q, const Fx* R, Fx* X, Fx* b) {
    const Fx zero{0, 0};
    for (int e = 0; e < N * N; e++) X[e] = zero;
    for (int i = N - 1; i >= 0; i--) {
        for (int k = 0; k < N; k++) b[k] = zero;
        for (int k = i; k < N; k++) {
            Fx s = zero;
            for (int p = i; p < k; p++) s = add(q, s, mul(q, R[p * N + k], true, b[p], false));
            const Fx e{k == i ? (int64_t(1) << q.f) : 0, 0};
            b[k] = divp(q, sub(q, e, s), R[k * N + k].re);
        }
        for (int k = i; k >= 0; k--) {
            Fx s = zero;
            for (int m = k + 1; m < N; m++) s = add(q, s, mul(q, R[k * N + m], false, FXP_XT(X, m, i), m > i));
            X[k * N + i] = divp(q, sub(q, b[k], s), R[k * N + k].re);
        }
    }
    mirror<N>(q, X);
}

template <int N>
__device__ void trimat(Q& q, const Fx* R, Fx* X, Fx* M) {
    const Fx zero{0, 0};
    for (int e = 0; e < N * N; e++) { X[e] = zero; M[e] = zero; }
    for (int i = 0; i < N; i++)
        for (int k = i; k >= 0; k--) {
            Fx s = zero;
            for (int m = k + 1; m <= i; m++) s = add(q, s, mul(q, R[k * N + m], false, M[m * N + i], false));
            const Fx e{k == i ? (int64_t(1) << q.f) : 0, 0};
            M[k * N + i] = divp(q, sub(q, e, s), R[k * N + k].re);
        }
    for (int i = 0; i < N; i++)
        for (int j = i; j < N; j++) {
            Fx s = zero;
            for (int p = j; p < N; p++) s = add(q, s, mul(q, M[i * N + p], false, M[j * N + p], true));
            X[i * N + j] = s;
        }
    mirror<N>(q, X);
}
#undef FXP_XT

constexpr int kThreads = 64;

template <int N>
__global__ void __launch_bounds__(kThreads)
k_fxp(int method, int m, int f, int64_t batch, const int64_t* __restrict__ A, int64_t* X,
      int32_t* __restrict__ info, int64_t* __restrict__ nsat)
{
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    Fx a[N * N], r[N * N], x[N * N], w[N * N];
    const int64_t* Ab = A + b * 2 * N * N;
    for (int e = 0; e < N * N; e++) a[e] = Fx{Ab[2 * e], Ab[2 * e + 1]};
    Q q{f, -(int64_t(1) << (m + f)), (int64_t(1) << (m + f)) - 1, 0};
    const int inf = chol<N>(q, a, r);
    if (inf == 0) {
        if (method == 0) proposed<N>(q, r, x);
        else if (method == 1) eqsolve<N>(q, r, x, w);
        else trimat<N>(q, r, x, w);
    } else {
        for (int e = 0; e < N * N; e++) x[e] = Fx{0, 0};
    }
    int64_t* Xb = X + b * 2 * N * N;
    for (int e = 0; e < N * N; e++) { Xb[2 * e] = x[e].re; Xb[2 * e + 1] = x[e].im; }
    info[b] = inf;
    nsat[b] = q.nsat;
}

template <int N>
static int launch(int method, int m, int f, int64_t batch, const int64_t* A, int64_t* X, int32_t* info,
                  int64_t* nsat, cudaStream_t s) {
    const int64_t blocks = (batch + kThreads - 1) / kThreads;
    k_fxp<N><<<unsigned(blocks), kThreads, 0, s>>>(method, m, f, batch, A, X, info, nsat);
    return int(cudaGetLastError());
}

}  // namespace fxp
}  // namespace hpdinv

using namespace hpdinv;

extern "C" int hpdinv_fxp_inv_batched(int method, int m, int f, int64_t batch, int n, const int64_t* A,
                                      int64_t* X, int32_t* info, int64_t* nsat, cudaStream_t stream) {
    if (method < 0 || method > 2) return -1;
    if (m < 1 || f < 1 || m + f > 40) return -2;
    if (batch < 0) return -4;
    if (n < 1 || n > 16) return -5;
    if (batch == 0) return 0;
    if (!A || reinterpret_cast<uintptr_t>(A) % 16) return -6;
    if (!X || reinterpret_cast<uintptr_t>(X) % 16) return -7;
    if (!info || reinterpret_cast<uintptr_t>(info) % 4) return -8;
    if (!nsat || reinterpret_cast<uintptr_t>(nsat) % 8) return -9;
    switch (n) {
#define HPDINV_FXP(NN) case NN: return fxp::launch<NN>(method, m, f, batch, A, X, info, nsat, stream);
        HPDINV_FXP(1) HPDINV_FXP(2) HPDINV_FXP(3) HPDINV_FXP(4) HPDINV_FXP(5) HPDINV_FXP(6)
        HPDINV_FXP(7) HPDINV_FXP(8) HPDINV_FXP(9) HPDINV_FXP(10) HPDINV_FXP(11) HPDINV_FXP(12)
        HPDINV_FXP(13) HPDINV_FXP(14) HPDINV_FXP(15) HPDINV_FXP(16)
#undef HPDINV_FXP
        default: return -5;
    }
}
