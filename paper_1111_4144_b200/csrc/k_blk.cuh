// k_blk.cuh -- one matrix per CTA, shared-memory resident, blocked into NB-row panels so that
// almost all of the work runs as register-tiled GEMM-shaped updates: the config-4 kernel
// (n = 64, complex128) and the config-5 kernel (n = 32, complex64, LDL).
//
// W (n x n, row stride n+1) holds one working matrix:
//   upper triangle: A -> U (the factor's rows: Cholesky R, LDL U = D R) -> X (in place, App. A.1);
//   lower triangle: R^T (w[j][k] = r_kj, written by the factor, read as columns of R) -> the
//                   mirror x_jk = conj(x_kj) of X (written by the inversion once R_KT is used).
// Factor (eqs. 3-4 / 10-11), panels K = [k0, k0+NB) in ascending order (Crout / left-looking):
//   F1  P_ij = a_ij - sum_{k<k0} conj(u_ki) r_kj  for i in K, j in [k0, n)     (GEMM, k ascending)
//   F2a one warp factors the NB x NB diagonal block of P (lane = column, right-looking)
//   F2b column-parallel panel solve of rows K for the columns j >= k0+NB (NB-step substitution)
// Proposed inversion (eqs. 20-24 / 25-29) in the blocked order of SURVEY App. A.2, panels
// from the bottom, T = [k0+NB, n) already inverted:
//   I1  C_kj = sum_{m in T} r_km x~_mj        (GEMM over the full Hermitian X_TT)
//   I2  x_kj = -(1/r_kk)(C_kj + sum_{m in K, m>k} r_km x_mj), j in T, rows k bottom-up
//   I3  V_kj = sum_{m in T} r_km conj(x_jm)   for k <= j in K (the x~_mj, m in T, of the block)
//   I4  one warp: the NB x NB diagonal block by the unblocked recursion with V added
// S5 copies W (= X, both halves, x_ji = conj(x_ij) bit for bit, Im x_ii = +0) to global memory.
#pragma once
#include "cplx.cuh"

namespace hpdinv {

template <typename T, int N, int NB, int NT, int RT>
struct BlkShape {
    static constexpr int LDW = N + 1;                 // odd row stride: column reads spread banks
    static constexpr int MINB = (NT >= 256) ? 3 : 1;  // 8-warp CTAs: registers for 3 CTAs/SM
    static constexpr int NBLK = N / NB;
    static constexpr int PR = NB / RT;                // row groups of a GEMM tile grid
    static constexpr int Q = NT / PR;                 // column groups
    static constexpr int CT = (N - NB + Q - 1) / Q;   // max columns per thread (panel width <= n - NB)
    // lookahead (NT >= 64): one warp runs the serial diagonal-block phases, NT - 32 threads the
    // GEMM of the rest: QR column groups; CTD columns per lane of the diagonal block's F1;
    // CTR (F1 rest, width <= n - 2 NB) and CTL (I1 lookahead, width <= n - NB, a power of two
    // dividing NB) columns per thread
#ifdef HPDINV_BLK_NOLA
    static constexpr bool LA = false;
#else
    static constexpr bool LA = NT >= 64;
#endif
    static constexpr int QR = NT >= 64 ? (NT - 32) / PR : 1;
    static constexpr int CTD = (NB + (32 / PR) - 1) / (32 / PR);
    static constexpr int CTR = (N - 2 * NB + QR - 1) / QR > 0 ? (N - 2 * NB + QR - 1) / QR : 1;
    static constexpr int CTL0 = (N - NB + QR - 1) / QR;
    static constexpr int CTL = CTL0 <= 1 ? 1 : CTL0 <= 2 ? 2 : CTL0 <= 4 ? 4 : 8;
    static constexpr size_t w_bytes = size_t(N) * LDW * sizeof(cplx<T>);
    static constexpr size_t v_off = ((w_bytes + 15) / 16) * 16;                 // V (NB x NB)
    static constexpr size_t s_off = v_off + size_t(NB) * NB * sizeof(cplx<T>);  // 1/r_kk, d_k
    static constexpr size_t smem_bytes = s_off + 2 * N * sizeof(T) + 16;
    static_assert(N % NB == 0 && NB <= 32 && NT % 32 == 0 && NB % RT == 0 && NT % PR == 0, "shape");
    static_assert(N - NB <= NT, "one thread per trailing column");
};

namespace blk {
#ifdef HPDINV_BLK_PROF
__device__ unsigned long long g_prof[2][16];   // per-phase cycles, summed over CTAs, of lane 0 of
                                               // [0] the serial warp and [1] the next warp
#define BLK_PHASE(id)                                             \
    do {                                                          \
        if (prof_on_) {                                           \
            const long long t_ = clock64();                       \
            prof_[prof_cur_] += t_ - prof_t_;                     \
            prof_t_ = t_;                                         \
            prof_cur_ = (id);                                     \
        }                                                         \
    } while (0)
#else
#define BLK_PHASE(id) do {} while (0)
#endif
__device__ __forceinline__ void cp_async_elem(void* dst, const void* src, int bytes) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
template <typename T> __device__ __forceinline__ cplx<T> shfl_c(cplx<T> v, int src) {
    return mk<T>(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// F1 (factor panel GEMM): for rows i = k0 + RT*p + r and columns j = k0 + q*CTT + c < n,
//   W[i][j] = a_ij - sum_{k<k0} conj(u_ki) r_kj      (u_ki = W[k][i] upper, r_kj = W[j][k] lower)
// fp64 subtracts term by term in k order (as written in eqs. 3-4); fp32 accumulates the sum with
// packed FFMA2 (split accumulator) and subtracts it once.
template <typename T, int N, int LDW, int RT, int CTT>
__device__ __forceinline__ void f1(cplx<T>* W, int k0, int p, int q, int c0 = -1, int cend = N) {
    using V = cplx<T>;
    if (c0 < 0) c0 = k0;
    if (c0 + q * CTT >= cend) return;
    int jc[CTT];
#pragma unroll
    for (int c = 0; c < CTT; c++) { const int j = c0 + q * CTT + c; jc[c] = j < cend ? j : cend - 1; }
    const int i0 = k0 + RT * p;
    if constexpr (sizeof(T) == 4) {
        SAcc<T> acc[RT][CTT];
#pragma unroll
        for (int r = 0; r < RT; r++)
#pragma unroll
            for (int c = 0; c < CTT; c++) sacc_zero(acc[r][c]);
#pragma unroll 2
        for (int k = 0; k < k0; k++) {
            V u[RT];
#pragma unroll
            for (int r = 0; r < RT; r++) u[r] = W[k * LDW + i0 + r];
#pragma unroll
            for (int c = 0; c < CTT; c++) {
                const V x = W[jc[c] * LDW + k];
#pragma unroll
                for (int r = 0; r < RT; r++) smac(acc[r][c], u[r], x);
            }
        }
#pragma unroll
        for (int c = 0; c < CTT; c++) {
            if (c0 + q * CTT + c < cend) {
#pragma unroll
                for (int r = 0; r < RT; r++) {
                    const V sv = sval_conjr(acc[r][c]);          // sum conj(u_ki) r_kj
                    V& w = W[(i0 + r) * LDW + jc[c]];
                    w = mk<T>(w.x - sv.x, w.y - sv.y);
                }
            }
        }
    } else {
        V acc[RT][CTT];
#pragma unroll
        for (int r = 0; r < RT; r++)
#pragma unroll
            for (int c = 0; c < CTT; c++) acc[r][c] = W[(i0 + r) * LDW + jc[c]];
#pragma unroll 2
        for (int k = 0; k < k0; k++) {
            V u[RT];
#pragma unroll
            for (int r = 0; r < RT; r++) u[r] = W[k * LDW + i0 + r];
#pragma unroll
            for (int c = 0; c < CTT; c++) {
                const V x = W[jc[c] * LDW + k];
#pragma unroll
                for (int r = 0; r < RT; r++) cfms_conj(acc[r][c], u[r], x);
            }
        }
#pragma unroll
        for (int c = 0; c < CTT; c++)
            if (c0 + q * CTT + c < cend) {
#pragma unroll
                for (int r = 0; r < RT; r++) W[(i0 + r) * LDW + jc[c]] = acc[r][c];
            }
    }
}

// I1 (inversion panel GEMM): for rows k = k0 + RT*p + r and columns j = t0 + q*CTT + c < n,
//   W[k][j] = C_kj = sum_{m=t0}^{n-1} r_km x~_mj   (r_km = W[m][k] lower, x~_mj = W[m][j] full X_TT)
// (it reads rows T only and writes rows K)
template <typename T, int N, int LDW, int RT, int CTT>
__device__ __forceinline__ void i1(cplx<T>* W, int k0, int t0, int p, int q, int c0 = -1, int mlo = -1) {
    using V = cplx<T>;
    if (c0 < 0) c0 = t0;
    if (c0 + q * CTT >= N) return;
    // inner range: m in [mlo, N) (default T); the lookahead passes columns of the block just
    // inverted with m in T only (their m in K terms wait for X_KK)
    if (mlo < 0) mlo = t0;
    int jc[CTT];
#pragma unroll
    for (int c = 0; c < CTT; c++) { const int j = c0 + q * CTT + c; jc[c] = j < N ? j : N - 1; }
    const int kr = k0 + RT * p;
    V cv[RT][CTT];
    if constexpr (sizeof(T) == 4) {
        SAcc<T> acc[RT][CTT];
#pragma unroll
        for (int r = 0; r < RT; r++)
#pragma unroll
            for (int c = 0; c < CTT; c++) sacc_zero(acc[r][c]);
#pragma unroll 2
        for (int m = mlo; m < N; m++) {
            V rk[RT];
#pragma unroll
            for (int r = 0; r < RT; r++) rk[r] = W[m * LDW + kr + r];
#pragma unroll
            for (int c = 0; c < CTT; c++) {
                const V x = W[m * LDW + jc[c]];
#pragma unroll
                for (int r = 0; r < RT; r++) smac(acc[r][c], rk[r], x);
            }
        }
#pragma unroll
        for (int r = 0; r < RT; r++)
#pragma unroll
            for (int c = 0; c < CTT; c++) cv[r][c] = sval(acc[r][c]);
    } else {
#pragma unroll
        for (int r = 0; r < RT; r++)
#pragma unroll
            for (int c = 0; c < CTT; c++) cv[r][c] = czero<T>();
#pragma unroll 2
        for (int m = mlo; m < N; m++) {
            V rk[RT];
#pragma unroll
            for (int r = 0; r < RT; r++) rk[r] = W[m * LDW + kr + r];
#pragma unroll
            for (int c = 0; c < CTT; c++) {
                const V x = W[m * LDW + jc[c]];
#pragma unroll
                for (int r = 0; r < RT; r++) cfma(cv[r][c], rk[r], x);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < CTT; c++)
        if (c0 + q * CTT + c < N) {
#pragma unroll
            for (int r = 0; r < RT; r++) W[(kr + r) * LDW + jc[c]] = cv[r][c];
        }
}
}  // namespace blk

template <typename T, int N, int NB, bool LDL, int NT, int RT>
__global__ void __launch_bounds__(NT, BlkShape<T, N, NB, NT, RT>::MINB)
k_blk(int64_t batch, const cplx<T>* __restrict__ A, int64_t sAm, int64_t sAe,
      cplx<T>* X, int64_t sXm, int64_t sXe, int32_t* __restrict__ info)
{
    using Sh = BlkShape<T, N, NB, NT, RT>;
    using V = cplx<T>;
    constexpr int LDW = Sh::LDW, PR = Sh::PR, Q = Sh::Q, CT = Sh::CT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* W = reinterpret_cast<V*>(smem_raw);
    V* Vs = reinterpret_cast<V*>(smem_raw + Sh::v_off);                          // V_kj of I3
    T* invs = reinterpret_cast<T*>(smem_raw + Sh::s_off);                        // 1/r_kk or 1/d_k
    T* dgs = invs + N;                                                           // LDL: d_k
    __shared__ int s_inf;
#define WE(i, j) W[(i) * LDW + (j)]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // the warp that runs the serial diagonal-block phases rotates with the CTA index, so the
    // co-resident CTAs' serial warps sit on different SM sub-partitions (warp w -> SMSP w % 4)
    const int swarp = int(blockIdx.x % unsigned(NT / 32));
    const int64_t b = blockIdx.x;
    const V* Ab = A + b * sAm;

#ifdef HPDINV_BLK_PROF
    long long prof_[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};   // F1 F2a F2b I1 I2 I3 I4 S5 - S1
    long long prof_t_ = clock64();
    int prof_cur_ = 9;                                  // 9 = S1 (load)
    const int prof_role_ = (warp == swarp) ? 0 : 1;
    const bool prof_on_ = lane == 0 && (warp == swarp || warp == (swarp + 1) % (NT / 32));
#endif
    // ------------------------------------------------------------------ S1: upper(A) -> W
    for (int e = tid; e < N * N; e += NT) {
        const int i = e / N, j = e - i * N;
        if (j >= i) blk::cp_async_elem(&WE(i, j), Ab + int64_t(e) * sAe, int(sizeof(V)));
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    if (tid == 0) s_inf = 0;
    __syncthreads();

    // GEMM tile of a thread: rows k0 + RT*p + r, columns c0 + q*ct + c (ct = panel width / Q)
    const int p = tid % PR, q = tid / PR;

    // ============================================================== factorisation, panels up
#pragma unroll 1
    for (int k0 = 0; k0 < N; k0 += NB) {
        BLK_PHASE(0);
        // ---- F1: P = A_K,[k0,n) - U_{<k0,K}^H R_{<k0,[k0,n)}  (k ascending, as in eqs. 3-4)
        if constexpr (Sh::LA) {
            // lookahead: the serial warp computes the diagonal block of P and factors it (F2a)
            // while the other warps compute the rest of the panel (nothing below depends on it)
            // (computing the diagonal block's F1 by all warps first, with split chains, measured
            // slower: the extra barrier costs more than the serial warp's longer chains)
            if (warp == swarp) {
                if (k0 > 0) blk::f1<T, N, LDW, RT, Sh::CTD>(W, k0, lane % PR, lane / PR, k0, k0 + NB);
                __syncwarp();
            } else if (k0 > 0 && k0 + NB < N) {
                const int rt = tid - (warp > swarp ? 32 : 0), pr = rt % PR, qr = rt / PR;
                const int ct = (N - k0 - NB + Sh::QR - 1) / Sh::QR;
                if (ct == 1) blk::f1<T, N, LDW, RT, 1>(W, k0, pr, qr, k0 + NB, N);
                else blk::f1<T, N, LDW, RT, Sh::CTR>(W, k0, pr, qr, k0 + NB, N);
            }
        } else {
            if (k0 > 0) {
                const int ct = (N - k0 + Q - 1) / Q;     // columns per thread for this panel width
                if (ct == 1) blk::f1<T, N, LDW, RT, 1>(W, k0, p, q);
                else if (ct == 2) blk::f1<T, N, LDW, RT, (CT >= 2 ? 2 : 1)>(W, k0, p, q);
                else blk::f1<T, N, LDW, RT, CT>(W, k0, p, q);
            }
            __syncthreads();
        }
        BLK_PHASE(1);
        // ---- F2a: diagonal block, warp swarp, lane l owns column k0 + l; row i of U is broadcast
        //      through shared memory, the pivot by one shuffle
        if (warp == swarp) {
            const int l = lane < NB ? lane : NB - 1;
            V pc[NB];
#pragma unroll
            for (int m = 0; m < NB; m++) pc[m] = WE(k0 + m, k0 + l);
            int bad_first = 0;
            T tnext = pc[0].x;
#pragma unroll
            for (int i = 0; i < NB; i++) {
                // the pivot comes from lane i's own update of its diagonal entry in the previous
                // step (u_{i-1,i} is its own value), bitwise what the shared-memory path gives,
                // so the serial chain skips the row exchange
                const T t = __shfl_sync(0xffffffffu, tnext, i);
                const bool bad = !(t > T(0));
                if (bad && bad_first == 0) bad_first = k0 + i + 1;
                const T tt = bad ? T(1) : t;                   // flagged: keep the arithmetic finite
                const T iv = LDL ? rcp_fast(tt) : rsqrt_fast(tt);
                const V r = cscale(pc[i], iv);                 // r_{k0+i, k0+l}, l > i
                const V u = LDL ? cscale(r, tt) : r;           // u = d r (LDL)
                if (i + 1 < NB) { V d = pc[i + 1]; cfms_conj(d, u, r); tnext = d.x; }
                if (lane == i) { invs[k0 + i] = iv; if (LDL) dgs[k0 + i] = tt; }
                if (lane > i && lane < NB) {
                    WE(k0 + i, k0 + lane) = u;                 // U row (upper)
                    WE(k0 + lane, k0 + i) = r;                 // R^T (lower)
                }
                __syncwarp();
                // right-looking update of the block: a_ml -= conj(u_im) r_il, i < m <= l
#pragma unroll
                for (int m = 0; m < NB; m++)
                    if (m > i) cfms_conj(pc[m], WE(k0 + i, k0 + m), r);
            }
            if (lane == 0 && bad_first && s_inf == 0) s_inf = bad_first;
        }
        __syncthreads();
        BLK_PHASE(2);
        // ---- F2b: rows K of the columns j >= k0 + NB (forward substitution through R_KK^H)
        {
            const int j = k0 + NB + tid;
            if (j < N) {
                V pc[NB];
#pragma unroll
                for (int m = 0; m < NB; m++) pc[m] = WE(k0 + m, j);
#pragma unroll
                for (int i = 0; i < NB; i++) {
                    const V r = cscale(pc[i], invs[k0 + i]);    // r_ij
                    const V u = LDL ? cscale(r, dgs[k0 + i]) : r;
                    WE(k0 + i, j) = u;
                    WE(j, k0 + i) = r;
#pragma unroll
                    for (int m = 0; m < NB; m++)
                        if (m > i) cfms_conj(pc[m], WE(k0 + i, k0 + m), r);   // -= conj(u_im) r_ij
                }
            }
        }
        __syncthreads();
    }

    const int inf = s_inf;
    if (inf == 0) {
    // ============================================================== inversion, panels down
#pragma unroll 1
    for (int k0 = N - NB; k0 >= 0; k0 -= NB) {
        const int t0 = k0 + NB;                       // T = [t0, n)
        BLK_PHASE(3);
        // ---- I1: C = R_KT X_TT into the upper K x T block (R_KT's upper copy is dead).  With
        //      the lookahead (NT >= 64) it was computed during the previous panel's I4, all but
        //      the terms m in K_prev = [t0, t0+NB) of the columns j in K_prev (added in I2)
        if constexpr (!Sh::LA) {
            if (t0 < N) {
                const int ct = (N - t0 + Q - 1) / Q;
                if (ct == 1) blk::i1<T, N, LDW, RT, 1>(W, k0, t0, p, q);
                else if (ct == 2) blk::i1<T, N, LDW, RT, (CT >= 2 ? 2 : 1)>(W, k0, t0, p, q);
                else blk::i1<T, N, LDW, RT, CT>(W, k0, t0, p, q);
            }
            __syncthreads();
        }
        BLK_PHASE(4);
        // ---- I2: rows K of the columns j in T, bottom-up (x_mj, m in K, stays in registers)
        V xk[NB];
        {
            const int j = t0 + tid;
            if (j < N) {
#pragma unroll
                for (int kk = NB - 1; kk >= 0; kk--) {
                    const int k = k0 + kk;
                    V s = WE(k, j);                                            // C_kj
                    // m descending: the term of the row just computed (m = kk+1) comes last, so
                    // the rest of the sum overlaps the previous row's latency
#pragma unroll
                    for (int m = NB - 1; m > kk; m--) cfma(s, WE(k0 + m, k), xk[m]);   // r_km x_mj
                    xk[kk] = LDL ? mk<T>(-s.x, -s.y) : cscale(s, -invs[k]);
                    WE(k, j) = xk[kk];
                }
            }
        }
        __syncthreads();
        BLK_PHASE(5);
        // ---- I3: V_kj = sum_{m in T} r_km conj(x_jm), k, j in K, into the scratch Vs; SPL
        //      adjacent threads split the sum over m and combine by shuffles
        if (t0 < N) {
            constexpr int SPL = (NT >= 2 * NB * NB) ? NT / (NB * NB) : 1;
            constexpr int OPS = NT / SPL;             // outputs per pass
            const int part = tid % SPL;
#pragma unroll 1
            for (int o = tid / SPL; o < NB * NB; o += OPS) {
                const int kk = o / NB, jj = o - kk * NB;
                V sv = czero<T>(), sv2 = czero<T>();                          // two chains
                int m = t0 + part;
                for (; m + SPL < N; m += 2 * SPL) {
                    cfma_cb(sv, WE(m, k0 + kk), WE(k0 + jj, m));
                    cfma_cb(sv2, WE(m + SPL, k0 + kk), WE(k0 + jj, m + SPL));
                }
                if (m < N) cfma_cb(sv, WE(m, k0 + kk), WE(k0 + jj, m));
                sv.x += sv2.x;
                sv.y += sv2.y;
#pragma unroll
                for (int off = 1; off < SPL; off <<= 1) {
                    sv.x += __shfl_xor_sync(0xffffffffu, sv.x, off);
                    sv.y += __shfl_xor_sync(0xffffffffu, sv.y, off);
                }
                if (part == 0) Vs[kk * NB + jj] = sv;
            }
        }
        __syncthreads();
        // mirror of the K x T rows (R^T_TK is no longer needed)
        {
            const int j = t0 + tid;
            if (j < N) {
#pragma unroll
                for (int kk = 0; kk < NB; kk++) WE(j, k0 + kk) = conjz(xk[kk]);
            }
        }
        if constexpr (Sh::LA) {
            __syncthreads();              // the lookahead below reads the mirror
            // lookahead I1 of the next panel K' = [k0-NB, k0), T' = [k0, n), by the warps that
            // do not run I4: columns j in T with m in T', columns j in K with m in T only
            if (warp != swarp && k0 > 0) {
                const int rt = tid - (warp > swarp ? 32 : 0), pr = rt % PR, qr = rt / PR;
                const int ct = (N - k0 + Sh::QR - 1) / Sh::QR;
                // CC columns per thread divides NB: each thread has one m range
                if (ct <= 1) blk::i1<T, N, LDW, RT, 1>(W, k0 - NB, k0, pr, qr, k0, k0 + qr < t0 ? t0 : k0);
                else if (ct <= 2) blk::i1<T, N, LDW, RT, 2>(W, k0 - NB, k0, pr, qr, k0, k0 + 2 * qr < t0 ? t0 : k0);
                else blk::i1<T, N, LDW, RT, Sh::CTL>(W, k0 - NB, k0, pr, qr, k0, k0 + Sh::CTL * qr < t0 ? t0 : k0);
            }
        }
        BLK_PHASE(6);
        // ---- I4: the diagonal block, warp swarp, lane l owns column k0 + l (full column in registers);
        //      row k of X goes to W at once (it overwrites the dead upper U row k) and the owner
        //      of column k reads it back as its lower part (the mirror) and forms x_kk
        if (warp == swarp) {
            const int l = lane < NB ? lane : NB - 1;
            const int j = k0 + l;
            V xc[NB];
#pragma unroll
            for (int m = 0; m < NB; m++) xc[m] = czero<T>();
#pragma unroll
            for (int kk = NB - 1; kk >= 0; kk--) {
                const int k = k0 + kk;
                const T ik = invs[k];
                V sv = (t0 < N) ? Vs[kk * NB + l] : czero<T>();                 // V_kj
#pragma unroll
                for (int m = NB - 1; m > kk; m--) cfma(sv, WE(k0 + m, k), xc[m]);   // r_km x~_mj
                const V xv = LDL ? mk<T>(-sv.x, -sv.y) : cscale(sv, -ik);
                if (lane > kk && lane < NB) { xc[kk] = xv; WE(k, j) = xv; }
                __syncwarp();
                if (lane == kk) {
                    T pd = (t0 < N) ? Vs[kk * NB + kk].x : T(0);                // Re V_kk
                    T pd2 = T(0);                                                // two chains
#pragma unroll
                    for (int m = 0; m < NB; m++) {
                        if (m > kk) {
                            const V xkm = WE(k, k0 + m);
                            if ((m - kk) & 1) pd = re_dot_conj(pd, WE(k0 + m, k), xkm);   // Re r_km conj(x_km)
                            else pd2 = re_dot_conj(pd2, WE(k0 + m, k), xkm);
                            xc[m] = conjz(xkm);
                        }
                    }
                    pd += pd2;
                    xc[kk] = mk<T>(LDL ? ik - pd : ik * (ik - pd), T(0));
                }
            }
            __syncwarp();
            if (lane < NB) {
#pragma unroll
                for (int m = 0; m < NB; m++) WE(k0 + m, j) = xc[m];            // column j, both halves
            }
        }
        __syncthreads();
        if constexpr (Sh::LA) {
            // lookahead: the terms m in K of the next panel's C_kj for the columns j in K (they
            // needed X_KK); k in K' = [k0-NB, k0)
            if (k0 > 0) {
                for (int o = tid; o < NB * NB; o += NT) {
                    const int k = k0 - NB + o / NB, j = k0 + o % NB;
                    V sv = WE(k, j);
#pragma unroll
                    for (int m = 0; m < NB; m++) cfma(sv, WE(k0 + m, k), WE(k0 + m, j));
                    WE(k, j) = sv;
                }
            }
            __syncthreads();
        }
    }
    }

    BLK_PHASE(7);
    // ------------------------------------------------------------------ S5: store X
    V* Xb = X + b * sXm;
    const T nan = qnan<T>();
    for (int e = tid; e < N * N; e += NT) {
        const int i = e / N, j = e - i * N;
        V v = WE(i, j);
        if (inf) v = mk<T>(nan, nan);
        Xb[int64_t(e) * sXe] = v;
    }
    if (tid == 0) info[b] = inf;
#ifdef HPDINV_BLK_PROF
    BLK_PHASE(8);
    if (prof_on_)
        for (int i = 0; i < 10; i++) atomicAdd(&blk::g_prof[prof_role_][i], (unsigned long long)prof_[i]);
#endif
#undef WE
}

}  // namespace hpdinv
