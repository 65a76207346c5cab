// k_base.cuh -- the paper's two EXISTING inversion methods on the GPU,
// so the proposed method's operation-count advantage (Table 1) can be measured on
// B200 against them on the same inputs and kernel structure.  Both start from the same
// Cholesky factor (eqs. 3-4) and write the full X = A^-1 with the Hermitian mirror:
//   METHOD 2, equation solving (eq. 15): for columns i = N..1, forward
//     substitution R* b_i = e_i (eq. 6; rows k < i are structurally zero and skipped), then back
//     substitution R x_i = b_i (eq. 7) for the upper half, rows k = i..1, using
//     x_mi = conj(x_im) for m > i (columns m > i are already known);
//   METHOD 3, triangular matrix operations (eqs. 16-19): M = R^-1 by R m_i = e_i
//     (eq. 18; upper triangular, rows k <= i), then the upper half of X = M M* (eq. 19).
// Structural zeros are exploited in every dot product (SURVEY App. A.3 "full exploitation":
// equation solving 2/3 n^3, triangular ops 1/2 n^3 + O(n^2) vs the proposed 1/2 n^3).
//   k_base_reg: one matrix per thread, R and X packed in registers (c64 n <= 8, c128 n <= 6);
//   k_base_gen: one matrix per CTA in shared memory, any n <= 64 (correctness path; the serial
//               substitutions run on one thread).
#pragma once
#include "cplx.cuh"
#include "k_reg.cuh"

namespace hpdinv {

template <typename T, int N, int METHOD>
__global__ void __launch_bounds__(kRegThreads)
k_base_reg(int64_t batch, const cplx<T>* __restrict__ A, int64_t sAm, int64_t sAe,
           cplx<T>* X, int64_t sXm, int64_t sXe, int32_t* __restrict__ info)
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
    const int inf = reg_factor<T, N, false>(r, inv);

    V x[NU];                                            // upper half of X, packed
    if constexpr (METHOD == 2) {
#pragma unroll
        for (int i = N - 1; i >= 0; i--) {
            V bv[N];
#pragma unroll
            for (int k = 0; k < N; k++) {               // eq. (6), rows k >= i
                if (k < i) continue;
                V s = k == i ? mk<T>(T(1), T(0)) : czero<T>();
#pragma unroll
                for (int p = 0; p < N; p++)
                    if (p >= i && p < k) cfms_conj(s, r[upk(N, p, k)], bv[p]);
                bv[k] = cscale(s, inv[k]);
            }
#pragma unroll
            for (int k = N - 1; k >= 0; k--) {          // eq. (7), rows k <= i
                if (k > i) continue;
                V s = k < i ? czero<T>() : bv[k];       // b_k = 0 above row i (R* lower triangular)
#pragma unroll
                for (int m = 0; m < N; m++) {
                    if (m <= k) continue;
                    const V xmi = (m <= i) ? x[upk(N, m, i)] : conjz(x[upk(N, i, m)]);
                    cfms(s, r[upk(N, k, m)], xmi);
                }
                V v = cscale(s, inv[k]);
                if (k == i) v.y = T(0);                 // x_ii is real (R4)
                x[upk(N, k, i)] = v;
            }
        }
    } else {
        V mm[NU];                                       // M = R^-1, upper, packed
#pragma unroll
        for (int i = 0; i < N; i++)
#pragma unroll
            for (int k = N - 1; k >= 0; k--) {          // eq. (18), rows k <= i
                if (k > i) continue;
                V s = k == i ? mk<T>(T(1), T(0)) : czero<T>();
#pragma unroll
                for (int m = 0; m < N; m++)
                    if (m > k && m <= i) cfms(s, r[upk(N, k, m)], mm[upk(N, m, i)]);
                mm[upk(N, k, i)] = cscale(s, inv[k]);
            }
#pragma unroll
        for (int i = 0; i < N; i++)                     // eq. (19): x_ij = sum_{p>=j} m_ip conj(m_jp)
#pragma unroll
            for (int j = 0; j < N; j++) {
                if (j < i) continue;
                V s = czero<T>();
#pragma unroll
                for (int p = 0; p < N; p++)
                    if (p >= j) cfma_cb(s, mm[upk(N, i, p)], mm[upk(N, j, p)]);
                if (i == j) s.y = T(0);
                x[upk(N, i, j)] = s;
            }
    }

    V* Xb = X + b * sXm;
    const T nan = qnan<T>();
#pragma unroll
    for (int i = 0; i < N; i++)
#pragma unroll
        for (int j = 0; j < N; j++) {
            V v = (i <= j) ? x[upk(N, i, j)] : conjz(x[upk(N, j, i)]);
            if (inf) v = mk<T>(nan, nan);
            Xb[int64_t(i * N + j) * sXe] = v;
        }
    info[b] = inf;
}

constexpr int kBaseGenThreads = 64;

template <typename T>
__host__ __device__ constexpr size_t base_gen_smem_bytes(int n) {
    return 2 * size_t(n) * n * sizeof(cplx<T>) + size_t(n) * sizeof(cplx<T>) + size_t(n) * sizeof(T);
}

template <typename T, int METHOD>
__global__ void __launch_bounds__(kBaseGenThreads)
k_base_gen(int64_t batch, int n, const cplx<T>* __restrict__ A, int64_t sAm, int64_t sAe,
           cplx<T>* X, int64_t sXm, int64_t sXe, int32_t* __restrict__ info)
{
    using V = cplx<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* R = reinterpret_cast<V*>(smem_raw);               // n*n, upper used
    V* W = R + n * n;                                     // X (eqsolve) or M (trimat), n*n
    V* bv = W + n * n;                                    // n
    T* inv = reinterpret_cast<T*>(bv + n);
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
        if (tid == 0) s_info = 0;
        __syncthreads();
        for (int i = 0; i < n; i++) {                    // Cholesky, eqs. (3)-(4)
            if (tid == 0) {
                T t = R[i * n + i].x;
                for (int k = 0; k < i; k++) {
                    const V rk = R[k * n + i];
                    t -= fma(rk.x, rk.x, rk.y * rk.y);
                }
                if (!(t > T(0)) && s_info == 0) s_info = i + 1;
                const T rr = sqrt_rn(t);
                R[i * n + i] = mk<T>(rr, T(0));
                inv[i] = rcp_rn(rr);
            }
            __syncthreads();
            for (int j = i + 1 + tid; j < n; j += blockDim.x) {
                V s = R[i * n + j];
                for (int k = 0; k < i; k++) cfms_conj(s, R[k * n + i], R[k * n + j]);
                R[i * n + j] = cscale(s, inv[i]);
            }
            __syncthreads();
        }
        if (tid == 0) {
            if constexpr (METHOD == 2) {
                for (int i = n - 1; i >= 0; i--) {
                    for (int k = i; k < n; k++) {
                        V s = k == i ? mk<T>(T(1), T(0)) : czero<T>();
                        for (int p = i; p < k; p++) cfms_conj(s, R[p * n + k], bv[p]);
                        bv[k] = cscale(s, inv[k]);
                    }
                    for (int k = i; k >= 0; k--) {
                        V s = k < i ? czero<T>() : bv[k];
                        for (int m = k + 1; m < n; m++) {
                            const V xmi = (m <= i) ? W[m * n + i] : conjz(W[i * n + m]);
                            cfms(s, R[k * n + m], xmi);
                        }
                        V v = cscale(s, inv[k]);
                        if (k == i) v.y = T(0);
                        W[k * n + i] = v;
                    }
                }
            } else {
                for (int i = 0; i < n; i++)
                    for (int k = i; k >= 0; k--) {
                        V s = k == i ? mk<T>(T(1), T(0)) : czero<T>();
                        for (int m = k + 1; m <= i; m++) cfms(s, R[k * n + m], W[m * n + i]);
                        W[k * n + i] = cscale(s, inv[k]);
                    }
                // X = M M* overwrites R's upper half (R is no longer needed)
                for (int i = 0; i < n; i++)
                    for (int j = i; j < n; j++) {
                        V s = czero<T>();
                        for (int p = j; p < n; p++) cfma_cb(s, W[i * n + p], W[j * n + p]);
                        if (i == j) s.y = T(0);
                        R[i * n + j] = s;
                    }
            }
        }
        __syncthreads();
        const V* Xs = METHOD == 2 ? W : R;
        const int inf = s_info;
        const T nan = qnan<T>();
        V* Xb = X + b * sXm;
        for (int e = tid; e < n * n; e += blockDim.x) {
            const int i = e / n, j = e - i * n;
            V v = (i <= j) ? Xs[i * n + j] : conjz(Xs[j * n + i]);
            if (inf) v = mk<T>(nan, nan);
            Xb[int64_t(e) * sXe] = v;
        }
        if (tid == 0) info[b] = inf;
        __syncthreads();
    }
}

}  // namespace hpdinv
