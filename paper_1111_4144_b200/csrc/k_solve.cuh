// k_solve.cuh -- batched HPD linear solve A x = y with the same factorisation (SURVEY §8(f)
// row f1): Cholesky eqs. (5)-(7), P:49-61 -- R* b = y by forward substitution, then R x = b
// by back substitution -- and LDL eqs. (12)-(14), P:87-99 -- R* D b = y, then R x = b with R
// unit upper.  A is read exactly as by the inversion (upper triangle, Im a_ii ignored); the
// factor is formed on chip and never stored.
//
//   k_solve_reg: one system per thread, the packed upper triangle in registers (n <= 8 c64,
//                n <= 6 c128); in the interleaved layout every load and store is coalesced
//                across the batch (the MIMO-equaliser shape, HBM bound);
//   k_solve_gen: one system per CTA in shared memory, any 1 <= n <= 64 (correctness path).
//
// info as for the inversion (first 1-based pivot with !(t > 0), LDL !(d > 0)); a flagged
// system's x is NaN.  Divisions by r_ii / d_i are multiplications by the reciprocal (R9).
#pragma once
#include "cplx.cuh"
#include "k_reg.cuh"

namespace hpdinv {

constexpr int kSolveThreads = 128;

template <typename T, int N, bool LDL>
__global__ void __launch_bounds__(kSolveThreads)
k_solve_reg(int64_t batch, const cplx<T>* __restrict__ A, int64_t sAm, int64_t sAe,
            const cplx<T>* __restrict__ Y, int64_t sYm, int64_t sYe,
            cplx<T>* Xv, int64_t sXm, int64_t sXe, int32_t* __restrict__ info)
{
    using V = cplx<T>;
    constexpr int NU = N * (N + 1) / 2;
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= batch) return;

    V r[NU];
    T inv[N];
    const V* Ab = A + b * sAm;
#pragma unroll
    for (int i = 0; i < N; i++)
#pragma unroll
        for (int j = 0; j < N; j++)
            if (j >= i) {
                V v = __ldg(Ab + int64_t(i * N + j) * sAe);
                if (i == j) v.y = T(0);
                r[upk(N, i, j)] = v;
            }
    V v[N];
    const V* Yb = Y + b * sYm;
#pragma unroll
    for (int i = 0; i < N; i++) v[i] = __ldg(Yb + int64_t(i) * sYe);

    const int inf = reg_factor<T, N, LDL>(r, inv);     // eqs. (3)-(4) / (10)-(11), in place

    // eq. (6) / (13): forward substitution, b_k = (y_k - sum_{p<k} conj(r_pk) w_p) / r_kk,
    // w_p = b_p (Cholesky) or d_p b_p (LDL, d_p on the diagonal of r)
    V w[N];
#pragma unroll
    for (int k = 0; k < N; k++) {
        V s = v[k];
#pragma unroll
        for (int p = 0; p < N; p++)
            if (p < k) cfms_conj(s, r[upk(N, p, k)], w[p]);
        v[k] = cscale(s, inv[k]);                       // b_k
        w[k] = LDL ? cscale(v[k], r[upk(N, k, k)].x) : v[k];
    }
    // eq. (7) / (14): back substitution, x_k = (b_k - sum_{m>k} r_km x_m) / r_kk (LDL: unit)
#pragma unroll
    for (int k = N - 1; k >= 0; k--) {
        V s = v[k];
#pragma unroll
        for (int m = 0; m < N; m++)
            if (m > k) cfms(s, r[upk(N, k, m)], v[m]);
        v[k] = LDL ? s : cscale(s, inv[k]);
    }

    V* Xb = Xv + b * sXm;
    const T nan = qnan<T>();
#pragma unroll
    for (int i = 0; i < N; i++) Xb[int64_t(i) * sXe] = inf ? mk<T>(nan, nan) : v[i];
    info[b] = inf;
}

constexpr int kSolveGenThreads = 64;

template <typename T>
__host__ __device__ constexpr size_t solve_gen_smem_bytes(int n) {
    return size_t(n) * n * sizeof(cplx<T>) + 2 * size_t(n) * sizeof(cplx<T>) + size_t(n) * sizeof(T);
}

template <typename T, bool LDL>
__global__ void __launch_bounds__(kSolveGenThreads)
k_solve_gen(int64_t batch, int n, const cplx<T>* __restrict__ A, int64_t sAm, int64_t sAe,
            const cplx<T>* __restrict__ Y, int64_t sYm, int64_t sYe,
            cplx<T>* Xv, int64_t sXm, int64_t sXe, int32_t* __restrict__ info)
{
    using V = cplx<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* R = reinterpret_cast<V*>(smem_raw);               // n*n, upper used; LDL: d_k on R[k][k].x
    V* bv = R + n * n;                                    // b, then x
    V* wv = bv + n;                                       // w_p = b_p or d_p b_p
    T* inv = reinterpret_cast<T*>(wv + n);                // 1/r_kk or 1/d_k
    __shared__ int s_info;
    const int tid = threadIdx.x;

    for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
        const V* Ab = A + b * sAm;
        for (int e = tid; e < n * n; e += blockDim.x) {
            const int i = e / n, j = e - i * n;
            if (j >= i) {
                V v = Ab[e * sAe];
                if (i == j) v.y = T(0);
                R[e] = v;
            }
        }
        for (int i = tid; i < n; i += blockDim.x) bv[i] = Y[b * sYm + int64_t(i) * sYe];
        if (tid == 0) s_info = 0;
        __syncthreads();

        // factorisation, row i at a time (eqs. 3-4 / 10-11), threads parallel over j
        for (int i = 0; i < n; i++) {
            if (tid == 0) {
                T t = R[i * n + i].x;
                for (int k = 0; k < i; k++) {
                    const V rk = R[k * n + i];
                    const T mag = fma(rk.x, rk.x, rk.y * rk.y);
                    t = LDL ? fma(-R[k * n + k].x, mag, t) : t - mag;
                }
                if (!(t > T(0)) && s_info == 0) s_info = i + 1;
                if (LDL) {
                    R[i * n + i] = mk<T>(t, T(0));
                    inv[i] = rcp_rn(t);
                } else {
                    const T rr = sqrt_rn(t);
                    R[i * n + i] = mk<T>(rr, T(0));
                    inv[i] = rcp_rn(rr);
                }
            }
            __syncthreads();
            for (int j = i + 1 + tid; j < n; j += blockDim.x) {
                V s = R[i * n + j];
                for (int k = 0; k < i; k++) {
                    V rki = R[k * n + i];
                    if (LDL) rki = cscale(rki, R[k * n + k].x);
                    cfms_conj(s, rki, R[k * n + j]);
                }
                R[i * n + j] = cscale(s, inv[i]);
            }
            __syncthreads();
        }

        // eq. (6) / (13) then eq. (7) / (14): O(n^2) substitutions, one thread per row update
        for (int k = 0; k < n; k++) {
            if (tid == 0) {
                V s = bv[k];
                for (int p = 0; p < k; p++) cfms_conj(s, R[p * n + k], wv[p]);
                bv[k] = cscale(s, inv[k]);
                wv[k] = LDL ? cscale(bv[k], R[k * n + k].x) : bv[k];
            }
        }
        if (tid == 0) {
            for (int k = n - 1; k >= 0; k--) {
                V s = bv[k];
                for (int m = k + 1; m < n; m++) cfms(s, R[k * n + m], bv[m]);
                bv[k] = LDL ? s : cscale(s, inv[k]);
            }
        }
        __syncthreads();
        const int inf = s_info;
        const T nan = qnan<T>();
        for (int i = tid; i < n; i += blockDim.x)
            Xv[b * sXm + int64_t(i) * sXe] = inf ? mk<T>(nan, nan) : bv[i];
        if (tid == 0) info[b] = inf;
        __syncthreads();
    }
}

}  // namespace hpdinv
