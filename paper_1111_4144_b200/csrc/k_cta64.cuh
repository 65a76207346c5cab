// k_cta64.cuh -- one matrix per CTA (128 threads), n = 64, shared-memory resident, blocked
// into two 32-row blocks so that most of the work runs as register-tiled GEMM-shaped updates
// (SURVEY App. A.2).  The config-4 kernel (complex128, "one matrix per CTA", BASELINE.json).
//
// Shared memory holds one 64 x 64 working matrix M (row stride 65 elements to spread banks):
// the upper triangle starts as A, becomes R in place, and is then overwritten by X
// block by block; the strict lower triangle is scratch (C, W, and the conjugate half of X).
//
// Factorisation (eqs. 3-4 / 10-11, right-looking, blocks K0 = [0,32), K1 = [32,64)):
//   F1  warp 0 factors the 32x32 diagonal block of K0 (lane q owns column q);
//   F2  panel solve R_01 = R_00^-H A_01: 32 columns x 4 row-phases, 8 lanes... (shuffles);
//   F3  trailing update A'_11 -= R_01^H R_01 (LDL: R_01^H D_0 R_01), 2x4 register tiles;
//   F4  warp 0 factors A'_11.
// Proposed inversion (eqs. 20-24 / 25-29) in the blocked order of App. A.2:
//   I1  warp 0: rows 63..32 -> X_11 (the unblocked recursion, lane q owns column 32+q);
//   I2  C = R_01 X_11 (register tiles), stored transposed in the lower-left block;
//   I3  rows 31..0 of X_01: x_kj = -inv_k (C_kj + sum_{k<m<32} r_km x_mj), column-parallel;
//   I4  W = R_01 X_01^H (register tiles) into the lower triangle of block 00;
//   I5  warp 0: rows 31..0 of X_00 with the extra term W (warps 1-3 mirror X_01 meanwhile);
//   then M (= X, both halves, x_ji = conj(x_ij)) is stored.
#pragma once
#include "cplx.cuh"

namespace hpdinv {

constexpr int kCta64Threads = 128;

template <typename T>
struct Cta64Shape {
    static constexpr int N = 64, B = 32, LD = 65;
    static constexpr size_t smem_bytes = size_t(N) * LD * sizeof(cplx<T>)   // M
                                         + size_t(N) * sizeof(T)             // inv
                                         + size_t(B) * sizeof(cplx<T>)       // row buffer
                                         + 16;
};

namespace cta64 {

template <typename T> __device__ __forceinline__ cplx<T>& at(cplx<T>* M, int i, int j) {
    return M[i * Cta64Shape<T>::LD + j];
}

__device__ __forceinline__ float shfl_t(float v, int src, int width = 32) { return __shfl_sync(0xffffffffu, v, src, width); }
__device__ __forceinline__ double shfl_t(double v, int src, int width = 32) { return __shfl_sync(0xffffffffu, v, src, width); }
template <typename T> __device__ __forceinline__ cplx<T> shfl_c(cplx<T> v, int src, int width = 32) {
    return mk<T>(shfl_t(v.x, src, width), shfl_t(v.y, src, width));
}
template <typename T> __device__ __forceinline__ cplx<T> csel(bool p, cplx<T> a, cplx<T> b) {
    return mk<T>(p ? a.x : b.x, p ? a.y : b.y);
}

// F1 / F4: warp-level right-looking factorisation of the 32x32 diagonal block at k0.
// Lane q owns column k0+q (rows k0..k0+31 in registers).  Row i of R is written to M as soon
// as it is scaled; the owner of column i broadcasts its pivot by shuffle.  LDL keeps d_i on
// the diagonal of M (R itself is unit diagonal).  Returns the first failing local pivot + 1.
template <typename T, bool LDL>
__device__ int factor_block(cplx<T>* M, T* inv, int k0, int lane) {
    constexpr int B = Cta64Shape<T>::B;
    const int j = k0 + lane;
    cplx<T> a[B];
#pragma unroll
    for (int l = 0; l < B; l++) a[l] = (l <= lane) ? at<T>(M, k0 + l, j) : czero<T>();
    int inf = 0;
#pragma unroll
    for (int i = 0; i < B; i++) {
        const T t = (lane == i) ? a[i].x : T(1);       // only the owner's radicand matters
        T iv;
        if (LDL) iv = rcp_rn(t);
        else iv = rcp_rn(sqrt_rn(t));
        const int bad = __shfl_sync(0xffffffffu, int(!(t > T(0))), i);
        iv = shfl_t(iv, i);
        if (bad && inf == 0) inf = i + 1;
        if (lane == i) {
            inv[k0 + i] = iv;
            at<T>(M, k0 + i, k0 + i) = mk<T>(LDL ? t : sqrt_rn(t), T(0));
        }
        const cplx<T> u = a[i];
        const cplx<T> r = cscale(u, iv);
        a[i] = r;
        if (lane > i) at<T>(M, k0 + i, j) = r;
        __syncwarp();
#pragma unroll
        for (int l = 0; l < B; l++) {
            if (l > i) {
                const cplx<T> ril = at<T>(M, k0 + i, k0 + l);     // broadcast read
                cfms_conj(a[l], ril, LDL ? u : r);                // rows l > lane: dead storage
            }
        }
    }
    __syncwarp();
    return inf;
}

// I1 / I5: warp-level proposed inversion of the 32x32 diagonal block at k0 (rows k0+31..k0).
// Lane q owns the full column k0+q of X_KK in registers.  With HAS_W the extra term W_kq
// (sum over the already inverted trailing rows) is read from M: W_kq at (k0+q, k0+k) for k < q
// and at (k0+k, k0+k) for k == q.  Row k of X overwrites row k of R (dead after the row) and
// its conjugate goes to column k (below the diagonal).
template <typename T, bool LDL, bool HAS_W>
__device__ void invert_block(cplx<T>* M, const T* inv, cplx<T>* rowbuf, int k0, int lane) {
    constexpr int B = Cta64Shape<T>::B;
    const int j = k0 + lane;
    cplx<T> x[B];
#pragma unroll
    for (int m = 0; m < B; m++) x[m] = czero<T>();
#pragma unroll
    for (int k = B - 1; k >= 0; k--) {
        const T ik = inv[k0 + k];
        cplx<T> acc = czero<T>();
        if (HAS_W && lane > k) acc = at<T>(M, j, k0 + k);
#pragma unroll
        for (int m = 0; m < B; m++) {
            if (m > k) cfma(acc, at<T>(M, k0 + k, k0 + m), x[m]);
        }
        const cplx<T> xv = LDL ? mk<T>(-acc.x, -acc.y) : cscale(acc, -ik);
        x[k] = xv;                                    // dead unless lane > k (see k_lane.cuh)
        if (lane > k) rowbuf[lane] = conjz(xv);
        __syncwarp();
        if (lane == k) {
            T s = HAS_W ? at<T>(M, k0 + k, k0 + k).x : T(0);
#pragma unroll
            for (int m = 0; m < B; m++) {
                if (m > k) {
                    x[m] = rowbuf[m];                 // x_mk = conj(x_km)
                    const cplx<T> rkm = at<T>(M, k0 + k, k0 + m);
                    s = fma(rkm.x, x[m].x, s);
                    s = fma(-rkm.y, x[m].y, s);       // Re(r_km x_mk)
                }
            }
            const T xkk = LDL ? ik - s : ik * (ik - s);
            x[k] = mk<T>(xkk, T(0));
        }
        __syncwarp();
        // row k of X replaces row k of R; its conjugate replaces W_kq below the diagonal
        if (lane > k) {
            at<T>(M, k0 + k, j) = xv;
            at<T>(M, j, k0 + k) = conjz(xv);
        }
        if (lane == k) at<T>(M, j, j) = x[k];
        __syncwarp();
    }
}

// Register-tiled 32x32x32 product over shared memory:  Out(r, c) = sum_m P(r, m) Q(m, c) with
// r = r0 + {rg, rg+16}, c = c0 + {ct, ct+8, ct+16, ct+24}; rg = warp*4 + lane/8, ct = lane%8.
// The loads of one warp hit 4 distinct P rows and 8 consecutive Q columns: one wavefront each.
template <typename T, typename PF, typename QF, typename OF>
__device__ __forceinline__ void tile_gemm32(PF P, QF Q, OF out, int warp, int lane) {
    const int rg = warp * 4 + (lane >> 3), ct = lane & 7;
    cplx<T> acc[2][4];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int c = 0; c < 4; c++) acc[a][c] = czero<T>();
#pragma unroll 4
    for (int m = 0; m < 32; m++) {
        cplx<T> p[2], q[4];
#pragma unroll
        for (int a = 0; a < 2; a++) p[a] = P(rg + 16 * a, m);
#pragma unroll
        for (int c = 0; c < 4; c++) q[c] = Q(m, ct + 8 * c);
#pragma unroll
        for (int a = 0; a < 2; a++)
#pragma unroll
            for (int c = 0; c < 4; c++) cfma(acc[a][c], p[a], q[c]);
    }
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int c = 0; c < 4; c++) out(rg + 16 * a, ct + 8 * c, acc[a][c]);
}

}  // namespace cta64

template <typename T, bool LDL>
#ifndef HPDINV_CTA64_MINB
#define HPDINV_CTA64_MINB 3
#endif
__global__ void __launch_bounds__(kCta64Threads, HPDINV_CTA64_MINB)
k_cta64(int64_t batch, const cplx<T>* __restrict__ A, int64_t sAm, int64_t sAe,
        cplx<T>* X, int64_t sXm, int64_t sXe, int32_t* __restrict__ info)
{
    using S = Cta64Shape<T>;
    using namespace cta64;
    constexpr int N = S::N, B = S::B;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* M = reinterpret_cast<cplx<T>*>(smem_raw);
    T* inv = reinterpret_cast<T*>(M + N * S::LD);
    cplx<T>* rowbuf = reinterpret_cast<cplx<T>*>(inv + N);
    __shared__ int s_info;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
        // ---------------------------------------------------------------- load upper(A)
        const cplx<T>* Ab = A + b * sAm;
        for (int e = tid; e < N * N; e += kCta64Threads) {
            const int i = e >> 6, jj = e & 63;
            if (jj >= i) {
                cplx<T> v = Ab[int64_t(e) * sAe];
                if (i == jj) v.y = T(0);
                at<T>(M, i, jj) = v;
            }
        }
        if (tid == 0) s_info = 0;
        __syncthreads();

        // ------------------------------------------------------------ F1: factor block 00
        if (warp == 0) {
            const int f = factor_block<T, LDL>(M, inv, 0, lane);
            if (lane == 0 && f) s_info = f;
        }
        __syncthreads();

        // ------------------------------------ F2: R_01 = R_00^-H A_01 (forward substitution)
        // thread -> column j = 32 + warp*8 + lane/4, rows i = p + 4t (p = lane%4, t = 0..7)
        {
            const int j = B + warp * 8 + (lane >> 2), p = lane & 3;
            cplx<T> a[8];
#pragma unroll
            for (int t = 0; t < 8; t++) a[t] = at<T>(M, p + 4 * t, j);
#pragma unroll
            for (int s = 0; s < B; s++) {
                const int ts = s >> 2;
                const cplx<T> u = shfl_c<T>(a[ts], s & 3, 4);          // a'_sj from its owner
                const cplx<T> r = cscale(u, inv[s]);                    // r_sj
                if (p == (s & 3)) {
                    a[ts] = r;
                    at<T>(M, s, j) = r;
                }
#pragma unroll
                for (int t = 0; t < 8; t++) {
                    if (4 * t + 3 > s) {                                // static: rows > s exist
                        const int i = p + 4 * t;
                        const cplx<T> rsi = csel<T>(i > s, at<T>(M, s, i), czero<T>());
                        cfms_conj(a[t], rsi, LDL ? u : r);
                    }
                }
            }
        }
        __syncthreads();

        // ------------------------------ F3: A'_11 -= R_01^H R_01  (LDL: R_01^H D_0 R_01)
        tile_gemm32<T>(
            [&](int l, int k) {                       // conj(r_{k,32+l}) (LDL: times d_k)
                const cplx<T> v = at<T>(M, k, B + l);
                return LDL ? cscale(conjz(v), at<T>(M, k, k).x) : conjz(v);
            },
            [&](int k, int c) { return at<T>(M, k, B + c); },
            [&](int l, int c, cplx<T> v) {
                if (l <= c) {
                    cplx<T>& d = at<T>(M, B + l, B + c);
                    d = mk<T>(d.x - v.x, d.y - v.y);
                }
            },
            warp, lane);
        __syncthreads();

        // ------------------------------------------------------------ F4: factor block 11
        if (warp == 0) {
            const int f = factor_block<T, LDL>(M, inv, B, lane);
            if (lane == 0 && f && s_info == 0) s_info = B + f;
        }
        __syncthreads();

        // ------------------------------------------------------- I1: X_11 (rows 63..32)
        if (warp == 0) invert_block<T, LDL, false>(M, inv, rowbuf, B, lane);
        __syncthreads();

        // -------------------------- I2: C = R_01 X_11, stored as C_kj at (j, k), j >= 32
        tile_gemm32<T>(
            [&](int k, int m) { return at<T>(M, k, B + m); },
            [&](int m, int c) { return at<T>(M, B + m, B + c); },
            [&](int k, int c, cplx<T> v) { at<T>(M, B + c, k) = v; },
            warp, lane);
        __syncthreads();

        // ------------- I3: rows 31..0 of X_01: x_kj = -inv_k (C_kj + sum_{k<m<32} r_km x_mj)
        {
            const int j = B + warp * 8 + (lane >> 2), p = lane & 3;
            cplx<T> c[8];
#pragma unroll
            for (int t = 0; t < 8; t++) c[t] = at<T>(M, j, p + 4 * t);
#pragma unroll
            for (int s = B - 1; s >= 0; s--) {
                const int ts = s >> 2;
                const cplx<T> cs = shfl_c<T>(c[ts], s & 3, 4);
                const cplx<T> xs = LDL ? mk<T>(-cs.x, -cs.y) : cscale(cs, -inv[s]);
                if (p == (s & 3)) at<T>(M, j, s) = conjz(xs);              // X_10 = X_01^H
#pragma unroll
                for (int t = 0; t < 8; t++) {
                    if (4 * t < s) {                                       // static: rows < s exist
                        const int k = p + 4 * t;
                        const cplx<T> rks = csel<T>(k < s, at<T>(M, k, s), czero<T>());
                        cfma(c[t], rks, xs);
                    }
                }
            }
        }
        __syncthreads();

        // --------- I4: W = R_01 X_01^H (upper 32x32): W_kq at (q, k) for k < q, at (k, k) for k == q
        tile_gemm32<T>(
            [&](int k, int m) { return at<T>(M, k, B + m); },
            [&](int m, int q) { return at<T>(M, B + m, q); },          // conj(x_qm)
            [&](int k, int q, cplx<T> v) {
                if (k < q) at<T>(M, q, k) = v;
                else if (k == q) at<T>(M, k, k) = v;
            },
            warp, lane);
        __syncthreads();

        // -------------------- I5: X_00 (warp 0) while warps 1-3 mirror X_01 into the upper block
        if (warp == 0) {
            invert_block<T, LDL, true>(M, inv, rowbuf, 0, lane);
        } else {
            for (int e = tid - 32; e < B * B; e += kCta64Threads - 32) {
                const int k = e >> 5, jj = B + (e & 31);
                at<T>(M, k, jj) = conjz(at<T>(M, jj, k));
            }
        }
        __syncthreads();

        // ------------------------------------------------------------------ store X
        const bool failed = s_info != 0;
        cplx<T>* Xb = X + b * sXm;
        const T nan = qnan<T>();
        for (int e = tid; e < N * N; e += kCta64Threads) {
            const int i = e >> 6, jj = e & 63;
            cplx<T> v = at<T>(M, i, jj);
            if (failed) v = mk<T>(nan, nan);
            Xb[int64_t(e) * sXe] = v;
        }
        if (tid == 0) info[b] = s_info;
        __syncthreads();
    }
}

}  // namespace hpdinv
