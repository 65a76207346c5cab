// k_nh.cuh -- inversion of non-Hermitian matrices through the HPD path (SURVEY §8(f) row f2,
// P:135-141): A = D D* is Hermitian positive definite for nonsingular D; A^-1 = X comes from
// the Cholesky factor (eqs. 3-4) and the proposed inversion (eqs. 20-24); D^-1 = D* X.
// All three steps are fused in one launch, nothing but D in and D^-1 out crosses HBM.
//
//   k_nh_reg: one matrix per thread (c64 n <= 8, c128 n <= 6).  A's packed upper triangle is
//             accumulated column by column of D (a_ij += d_ip conj(d_jp)), so only one column
//             of D and the triangle are live; D^-1 is formed row by row, (D^-1)_ij =
//             sum_p conj(d_pi) x_pj, re-reading column i of D from the thread's shared-memory
//             copy (written during the first pass).
//   k_nh_gen: one matrix per CTA in shared memory, any n <= 64 (correctness path).
// info: the Cholesky info of A = DD* (0 <=> D numerically nonsingular); D^-1 NaN when flagged.
#pragma once
#include "cplx.cuh"
#include "k_reg.cuh"

namespace hpdinv {

template <typename T, int N>
__global__ void __launch_bounds__(kRegThreads)
k_nh_reg(int64_t batch, const cplx<T>* __restrict__ D, int64_t sDm, int64_t sDe,
         cplx<T>* Y, int64_t sYm, int64_t sYe, int32_t* __restrict__ info)
{
    using V = cplx<T>;
    constexpr int NU = N * (N + 1) / 2;
    const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    const V* Db = D + b * sDm;
    // D as read in the first pass, kept for the second in this thread's shared-memory column
    // (element e at Ds[e * blockDim.x]: a warp's 8- or 16-byte accesses are conflict-free)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* Ds = reinterpret_cast<V*>(smem_raw) + threadIdx.x;

    V r[NU];
#pragma unroll
    for (int e = 0; e < NU; e++) r[e] = czero<T>();
    {                                                   // A = D D*, p ascending (column p+1
        V c[N];                                         // fetched during the update with p)
#pragma unroll
        for (int i = 0; i < N; i++) {
            c[i] = __ldg(Db + int64_t(i * N) * sDe);
            Ds[(i * N) * kRegThreads] = c[i];
        }
#pragma unroll
        for (int p = 0; p < N; p++) {
            V cn[N];
            const int p1 = p + 1 < N ? p + 1 : p;
            if (p + 1 < N) {
#pragma unroll
                for (int i = 0; i < N; i++) {
                    cn[i] = __ldg(Db + int64_t(i * N + p1) * sDe);
                    Ds[(i * N + p1) * kRegThreads] = cn[i];
                }
            }
#pragma unroll
            for (int i = 0; i < N; i++)
#pragma unroll
                for (int j = 0; j < N; j++)
                    if (j >= i) cfma_cb(r[upk(N, i, j)], c[i], c[j]);
#pragma unroll
            for (int i = 0; i < N; i++) c[i] = cn[i];
        }
    }
#pragma unroll
    for (int i = 0; i < N; i++) r[upk(N, i, i)].y = T(0);   // a_ii real (R5: Im a_ii ignored)

    T inv[N];
    const int inf = reg_factor<T, N, false>(r, inv);
    reg_invert<T, N, false>(r, inv);                     // r = upper half of X = A^-1

    V* Yb = Y + b * sYm;
    const T nan = qnan<T>();
    // rows of D^-1 = D* X, i ascending; column i+1 of D is read (shared memory) while row i is
    // formed (fully unrolled: 0.37 -> 0.34 ms at cfg7 against rolled loops, despite 255 registers;
    // re-reading D from L2 instead of shared memory: 0.34 ms)
    V c[N];
#pragma unroll
    for (int p = 0; p < N; p++) c[p] = Ds[(p * N) * kRegThreads];                     // d_p0
#pragma unroll
    for (int i = 0; i < N; i++) {
        V cn[N];
        const int i1 = i + 1 < N ? i + 1 : i;
#pragma unroll
        for (int p = 0; p < N; p++) cn[p] = Ds[(p * N + i1) * kRegThreads];
#pragma unroll
        for (int j = 0; j < N; j++) {
            V s = czero<T>();
#pragma unroll
            for (int p = 0; p < N; p++) {
                const V xpj = (p <= j) ? r[upk(N, p, j)] : conjz(r[upk(N, j, p)]);
                cfma_cb(s, xpj, c[p]);                   // += x_pj conj(d_pi)
            }
            Yb[int64_t(i * N + j) * sYe] = inf ? mk<T>(nan, nan) : s;
        }
#pragma unroll
        for (int p = 0; p < N; p++) c[p] = cn[p];
    }
    info[b] = inf;
}

constexpr int kNhGenThreads = 64;

template <typename T>
__host__ __device__ constexpr size_t nh_gen_smem_bytes(int n) {
    return 3 * size_t(n) * n * sizeof(cplx<T>) + size_t(n) * sizeof(T);
}

template <typename T>
__global__ void __launch_bounds__(kNhGenThreads)
k_nh_gen(int64_t batch, int n, const cplx<T>* __restrict__ D, int64_t sDm, int64_t sDe,
         cplx<T>* Y, int64_t sYm, int64_t sYe, int32_t* __restrict__ info)
{
    using V = cplx<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* Ds = reinterpret_cast<V*>(smem_raw);              // D, n*n
    V* R = Ds + n * n;                                     // A -> R (upper)
    V* Xs = R + n * n;                                     // X (upper)
    T* inv = reinterpret_cast<T*>(Xs + n * n);
    __shared__ int s_info;
    const int tid = threadIdx.x;

    for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
        const V* Db = D + b * sDm;
        for (int e = tid; e < n * n; e += blockDim.x) Ds[e] = Db[e * sDe];
        if (tid == 0) s_info = 0;
        __syncthreads();
        for (int e = tid; e < n * n; e += blockDim.x) {  // A = D D*, upper
            const int i = e / n, j = e - i * n;
            if (j >= i) {
                V s = czero<T>();
                for (int p = 0; p < n; p++) cfma_cb(s, Ds[i * n + p], Ds[j * n + p]);
                if (i == j) s.y = T(0);
                R[e] = s;
            }
        }
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
        for (int k = n - 1; k >= 0; k--) {               // proposed inversion, eqs. (20)-(24)
            for (int j = k + 1 + tid; j < n; j += blockDim.x) {
                V s = czero<T>();
                for (int m = k + 1; m < n; m++) {
                    const V xmj = (m <= j) ? Xs[m * n + j] : conjz(Xs[j * n + m]);
                    cfma(s, R[k * n + m], xmj);
                }
                Xs[k * n + j] = cscale(s, -inv[k]);
            }
            __syncthreads();
            if (tid == 0) {
                T s = T(0);
                for (int m = k + 1; m < n; m++) s = re_dot_conj(s, R[k * n + m], Xs[k * n + m]);
                Xs[k * n + k] = mk<T>(inv[k] * (inv[k] - s), T(0));
            }
            __syncthreads();
        }
        const int inf = s_info;
        const T nan = qnan<T>();
        V* Yb = Y + b * sYm;
        for (int e = tid; e < n * n; e += blockDim.x) {  // D^-1 = D* X
            const int i = e / n, j = e - i * n;
            V s = czero<T>();
            for (int p = 0; p < n; p++) {
                const V xpj = (p <= j) ? Xs[p * n + j] : conjz(Xs[j * n + p]);
                cfma_cb(s, xpj, Ds[p * n + i]);
            }
            Yb[int64_t(e) * sYe] = inf ? mk<T>(nan, nan) : s;
        }
        if (tid == 0) info[b] = inf;
        __syncthreads();
    }
}

}  // namespace hpdinv
