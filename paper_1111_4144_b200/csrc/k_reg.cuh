// k_reg.cuh -- one matrix per thread, the whole upper triangle in registers (small n).
//
// Every loop is fully unrolled over the compile-time size N so the packed upper triangle
// r[] lives in registers.  The steps are exactly the hot path of SURVEY §8(a):
//   S1 load upper(A) (coalesced across the batch in the interleaved layout),
//   S2 Cholesky eqs. (3)-(4) / S2' LDL eqs. (10)-(11), in place,
//   S3 shortcut S = diag(1/r_ii) (eq. 24) / S~ = diag(1/d_i) (eq. 29) kept as N reciprocals,
//   S4 rows k = N..1 of the upper half of X (eqs. 22-24), row k of X overwriting row k of R,
//   S5 mirror x_ji = conj(x_ij) and store.
#pragma once
#include "cplx.cuh"

namespace hpdinv {

constexpr int kRegThreads = 128;

// S2 / S2': factorisation of the packed upper triangle r[] in place (eqs. 3-4 / 10-11; sums
// in k ascending as written); LDL keeps d_i on the diagonal.  inv[i] = 1/r_ii (1/d_i).
// Returns info: the first 1-based i with !(t_i > 0), else 0.
template <typename T, int N, bool LDL>
__device__ __forceinline__ int reg_factor(cplx<T> (&r)[N * (N + 1) / 2], T (&inv)[N]) {
    int inf = 0;
#pragma unroll
    for (int i = 0; i < N; i++) {
        cplx<T> w[N > 1 ? N - 1 : 1];
        T t = r[upk(N, i, i)].x;
#pragma unroll
        for (int k = 0; k < N; k++) {
            if (k >= i) continue;
            const cplx<T> rki = r[upk(N, k, i)];
            if (LDL) {
                const T dk = r[upk(N, k, k)].x;             // d_k stored on the diagonal
                w[k] = cscale(rki, dk);                     // w_k = d_k r_ki (conj applied below)
                t = fma(-w[k].x, rki.x, t);
                t = fma(-w[k].y, rki.y, t);
            } else {
                w[k] = rki;
                t = fma(-rki.x, rki.x, t);
                t = fma(-rki.y, rki.y, t);
            }
        }
        if (!(t > T(0)) && inf == 0) inf = i + 1;
        T iv;
        if (LDL) {
            iv = rcp_rn(t);
            r[upk(N, i, i)] = mk<T>(t, T(0));
        } else {
            const T rii = sqrt_rn(t);
            iv = rcp_rn(rii);
            r[upk(N, i, i)] = mk<T>(rii, T(0));
        }
        inv[i] = iv;
#pragma unroll
        for (int j = 0; j < N; j++) {
            if (j <= i) continue;
            cplx<T> s = r[upk(N, i, j)];
#pragma unroll
            for (int k = 0; k < N; k++)
                if (k < i) cfms_conj(s, w[k], r[upk(N, k, j)]);
            r[upk(N, i, j)] = cscale(s, iv);
        }
    }

    return inf;
}

// S3 / S4: the proposed inversion (eqs. 20-24 / 25-29), rows k = N-1..0, in place over the
// factor's packed upper triangle (row k of X overwrites row k of R, App. A.1); x_kk real (R4).
template <typename T, int N, bool LDL>
__device__ __forceinline__ void reg_invert(cplx<T> (&r)[N * (N + 1) / 2], const T (&inv)[N]) {
#pragma unroll
    for (int k = N - 1; k >= 0; k--) {
        cplx<T> t[N];
#pragma unroll
        for (int j = 0; j < N; j++) {
            if (j <= k) continue;
            cplx<T> s = czero<T>();
#pragma unroll
            for (int m = 0; m < N; m++) {
                if (m <= k) continue;
                const cplx<T> xmj = (m <= j) ? r[upk(N, m, j)] : conjz(r[upk(N, j, m)]);
                cfma(s, r[upk(N, k, m)], xmj);
            }
            t[j] = LDL ? mk<T>(-s.x, -s.y) : cscale(s, -inv[k]);
        }
        T s = T(0);
#pragma unroll
        for (int m = 0; m < N; m++)
            if (m > k) s = re_dot_conj(s, r[upk(N, k, m)], t[m]);
        const T xkk = LDL ? inv[k] - s : inv[k] * (inv[k] - s);
        r[upk(N, k, k)] = mk<T>(xkk, T(0));
#pragma unroll
        for (int j = 0; j < N; j++)
            if (j > k) r[upk(N, k, j)] = t[j];
    }

}

template <typename T, int N, bool LDL>
__global__ void __launch_bounds__(kRegThreads)
k_reg(int64_t batch, const cplx<T>* __restrict__ A, int64_t sAm, int64_t sAe,
      cplx<T>* X, int64_t sXm, int64_t sXe, int32_t* __restrict__ info)
{
    constexpr int NU = N * (N + 1) / 2;
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= batch) return;

    cplx<T> r[NU];
    T inv[N];
    const cplx<T>* Ab = A + b * sAm;
#pragma unroll
    for (int i = 0; i < N; i++)
#pragma unroll
        for (int j = 0; j < N; j++) {
            if (j >= i) {
                cplx<T> v = __ldg(Ab + int64_t(i * N + j) * sAe);
                if (i == j) v.y = T(0);
                r[upk(N, i, j)] = v;
            }
        }

    // ---- S2: factorisation
    const int inf = reg_factor<T, N, LDL>(r, inv);

    // ---- S3/S4: proposed inversion
    reg_invert<T, N, LDL>(r, inv);

    // ---- S5: mirror + store
    cplx<T>* Xb = X + b * sXm;
    const T nan = qnan<T>();
#pragma unroll
    for (int i = 0; i < N; i++)
#pragma unroll
        for (int j = 0; j < N; j++) {
            cplx<T> v = (i <= j) ? r[upk(N, i, j)] : conjz(r[upk(N, j, i)]);
            if (inf) v = mk<T>(nan, nan);
            Xb[int64_t(i * N + j) * sXe] = v;
        }
    info[b] = inf;
}

}  // namespace hpdinv
