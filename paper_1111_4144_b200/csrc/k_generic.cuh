// k_generic.cuh -- one matrix per CTA, shared-memory resident, any 1 <= n <= 64, any dtype,
// any accepted layout.  The correctness baseline of the library and the path for sizes that
// have no specialised kernel.  Rows of R are produced by eqs. (3)-(4) (LDL: (10)-(11)) with
// the threads of the CTA parallel over the column index j; the inversion runs rows k = n..1
// (eqs. 20-24 / 25-29, SURVEY App. A.1 order) with the threads parallel over j.
#pragma once
#include "cplx.cuh"

namespace hpdinv {

constexpr int kGenericThreads = 64;

template <typename T>
__host__ __device__ constexpr size_t generic_smem_bytes(int n) {
    return 2 * size_t(n) * n * sizeof(cplx<T>) + size_t(n) * sizeof(T);
}

template <typename T, bool LDL>
__global__ void __launch_bounds__(kGenericThreads)
k_generic(int64_t batch, int n, const cplx<T>* __restrict__ A, int64_t sAm, int64_t sAe,
          cplx<T>* X, int64_t sXm, int64_t sXe, int32_t* __restrict__ info)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* R = reinterpret_cast<cplx<T>*>(smem_raw);  // n*n, upper used; LDL: d_k on R[k][k].x
    cplx<T>* Xs = R + n * n;                             // n*n, upper used
    T* inv = reinterpret_cast<T*>(Xs + n * n);           // 1/r_kk (Cholesky) or 1/d_k (LDL)
    __shared__ int s_info;
    const int tid = threadIdx.x;

    for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
        const cplx<T>* Ab = A + b * sAm;
        for (int e = tid; e < n * n; e += blockDim.x) {
            int i = e / n, j = e - i * n;
            if (j >= i) {
                cplx<T> v = Ab[e * sAe];
                if (i == j) v.y = T(0);
                R[e] = v;
            }
        }
        if (tid == 0) s_info = 0;
        __syncthreads();

        // ---- factorisation, row i at a time
        for (int i = 0; i < n; i++) {
            if (tid == 0) {
                T t = R[i * n + i].x;
                for (int k = 0; k < i; k++) {
                    cplx<T> rk = R[k * n + i];
                    T mag = fma(rk.x, rk.x, rk.y * rk.y);
                    t = LDL ? fma(-R[k * n + k].x, mag, t) : t - mag;
                }
                if (!(t > T(0)) && s_info == 0) s_info = i + 1;
                if (LDL) {
                    R[i * n + i] = mk<T>(t, T(0));     // d_i (R itself is unit diagonal)
                    inv[i] = rcp_rn(t);
                } else {
                    T r = sqrt_rn(t);
                    R[i * n + i] = mk<T>(r, T(0));
                    inv[i] = rcp_rn(r);
                }
            }
            __syncthreads();
            for (int j = i + 1 + tid; j < n; j += blockDim.x) {
                cplx<T> s = R[i * n + j];
                for (int k = 0; k < i; k++) {
                    cplx<T> rki = R[k * n + i];
                    if (LDL) rki = cscale(rki, R[k * n + k].x);   // w_k = d_k r_ki (conj below)
                    cfms_conj(s, rki, R[k * n + j]);
                }
                R[i * n + j] = cscale(s, inv[i]);
            }
            __syncthreads();
        }

        // ---- proposed inversion: rows k = n-1..0 of the upper half of X
        for (int k = n - 1; k >= 0; k--) {
            for (int j = k + 1 + tid; j < n; j += blockDim.x) {
                cplx<T> s = czero<T>();
                for (int m = k + 1; m < n; m++) {
                    cplx<T> xmj = (m <= j) ? Xs[m * n + j] : conjz(Xs[j * n + m]);
                    cfma(s, R[k * n + m], xmj);
                }
                Xs[k * n + j] = LDL ? mk<T>(-s.x, -s.y) : cscale(s, -inv[k]);
            }
            __syncthreads();
            if (tid == 0) {
                T s = T(0);
                for (int m = k + 1; m < n; m++) s = re_dot_conj(s, R[k * n + m], Xs[k * n + m]);
                T xkk = LDL ? inv[k] - s : inv[k] * (inv[k] - s);
                Xs[k * n + k] = mk<T>(xkk, T(0));
            }
            __syncthreads();
        }

        // ---- mirror + store
        const bool failed = s_info != 0;
        cplx<T>* Xb = X + b * sXm;
        for (int e = tid; e < n * n; e += blockDim.x) {
            int i = e / n, j = e - i * n;
            cplx<T> v = (i <= j) ? Xs[i * n + j] : conjz(Xs[j * n + i]);
            if (failed) v = mk<T>(qnan<T>(), qnan<T>());
            Xb[e * sXe] = v;
        }
        if (tid == 0) info[b] = s_info;
        __syncthreads();
    }
}

}  // namespace hpdinv
