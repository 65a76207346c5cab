// k_dmma.cuh -- n = 64, complex128, Cholesky: one matrix per CTA (4 warps), the GEMM-shaped
// updates on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64) -- the config-4 kernel.
//
// Why DMMA: on B200 the FP64 DMMA path reaches 37.05 TF/s (tools/mma_peaks.cu,
// profiles/r02_mma_peaks.txt) against 33.4 for DFMA, on the same FP64 datapath, and one DMMA
// instruction carries 256 FMAs instead of 32: the blocked algorithm stops being bound by
// instruction issue, shared-memory operand traffic and register-bank conflicts (the round-1
// k_blk ran 48k warp instructions per matrix for 16k DFMA).
//
// Storage (shared memory, 36 KB per matrix): only the 36 UPPER 8 x 8 tiles (I <= J) of the
// working matrix, complex interleaved, 1 KB per tile; element (r, c) of a tile at 16-byte slot
// r*8 + (c ^ r) -- the 128-byte TMA swizzle, so S1 is 36 cp.async.bulk.tensor tile loads with
// one mbarrier.  Every fragment access pattern of the kernel is bank-conflict free in this
// layout (quarter-warp phases of the 16-byte accesses), provided the k index of a k-step s of
// the m8n8k4 MMA runs over the tile columns {s, 2+s, 4+s, 6+s}: lane t (q = t % 4) then holds
// k = 2q + s, which is exactly the column of its own accumulator element e = s -- so a
// conjugate-transposed operand X^H can be fed to the next MMA straight from the accumulator
// registers (I3 below).  Tile (I, J) holds A -> R (the factor, upper) -> X (in place,
// App. A.1); the diagonal tile holds R_KK in its upper half, then the FULL Hermitian X_KK.
//
// Factor (eqs. 3-4), panels K = 0..7 (left-looking: the sums of eqs. 3-4 over k < 8K at once):
//   F1  A_KJ -= sum_{P<K} R_PK^H R_PJ  for J >= K       (DMMA, accumulators start at A_KJ)
//   F2a warp 0: R_KK by the right-looking recursion of eqs. 3-4 on its accumulator registers
//       (pivots and rows broadcast by shuffles); info = first k with !(t_k > 0)
//   F2b warps 1-3: R_KJ = R_KK^-H A_KJ, the forward substitution of eq. 4 on the accumulator
//       registers (row i broadcast down the columns by shuffles)
// Proposed inversion (eqs. 20-24), panels K = 7..0, T = K+1..7:
//   I1  C_KJ = sum_{M in T} R_KM X~_MJ  for J in T    (DMMA; X~_MJ = X_JM^H read transposed)
//   I2  x_kj = -(1/r_kk)(C_kj + sum_{m in K, m>k} r_km x_mj), k = 7..0 (registers, shuffles)
//   I3  V = sum_{J in T} R_KJ X_KJ^H (DMMA, X^H from the accumulators), per-warp partials
//   I4  warp 0: X_KK by the recursion of eq. 23 with V_kj added (lane j owns column j; the row
//       gathered to the diagonal lane by shuffles is the mirror), x_kk real
// S5  every tile to global memory, lower tiles as the conjugate transpose (bitwise mirror).
#pragma once
#include <cuda.h>
#include "cplx.cuh"

namespace hpdinv {
namespace dm {

constexpr int N = 64;
constexpr int NTL = 8;                               // tiles per dimension
constexpr int NTILE = NTL * (NTL + 1) / 2;           // 36 upper tiles
constexpr int NT = 128;                              // threads per CTA (4 warps)
constexpr int TILE_B = 1024;
constexpr int OFF_V = NTILE * TILE_B;                // 4 per-warp V partials
constexpr int OFF_INV = OFF_V + 4 * TILE_B;          // 1/r_kk, 64 doubles
constexpr int OFF_BAR = OFF_INV + N * 8;             // mbarrier, info
constexpr int SMEM_USED = OFF_BAR + 16;
constexpr int SMEM = SMEM_USED + 1024;               // + alignment slack (TMA 128B swizzle: 1 KB)

__host__ __device__ constexpr int tidx(int I, int J) { return I * NTL - I * (I - 1) / 2 + (J - I); }
__device__ __forceinline__ int sw(int r, int c) { return r * 8 + (c ^ r); }

__device__ __forceinline__ double negd(double x) {   // sign flip on the integer pipe
    return __hiloint2double(__double2hiint(x) ^ int(0x80000000), __double2loint(x));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// complex 8x8 accumulator tile in the m8n8k4 C layout: lane t holds (t/4, 2(t%4) + e), e = 0, 1
struct CAcc { double r0, r1, i0, i1; };

__device__ __forceinline__ void czero(CAcc& c) { c.r0 = c.r1 = c.i0 = c.i1 = 0.0; }

// c += A B for one k-step: a = (ar, ai) the A fragment, nai = -ai, b = (br, bi) the B fragment
__device__ __forceinline__ void cmma(CAcc& c, double ar, double ai, double nai, double br, double bi) {
    dmma(c.r0, c.r1, ar, br);
    dmma(c.i0, c.i1, ar, bi);
    dmma(c.r0, c.r1, nai, bi);
    dmma(c.i0, c.i1, ai, br);
}

// fragment loads (element (re, im) as one 16-byte shared load):
//   fa: element (t/4, 2q+s) of the tile -- an A operand as stored, or a B operand transposed
//   fb: element (2q+s, t/4) of the tile -- a B operand as stored, or an A operand transposed
__device__ __forceinline__ double2 fa(const double2* tl, int lane, int s) {
    const int r = lane >> 2, c = 2 * (lane & 3) + s;
    return tl[sw(r, c)];
}
__device__ __forceinline__ double2 fb(const double2* tl, int lane, int s) {
    const int r = 2 * (lane & 3) + s, c = lane >> 2;
    return tl[sw(r, c)];
}

__device__ __forceinline__ void acc_load(CAcc& c, const double2* tl, int lane) {
    const int r = lane >> 2, c0 = 2 * (lane & 3);
    const double2 a = tl[sw(r, c0)], b = tl[sw(r, c0 + 1)];
    c.r0 = a.x; c.i0 = a.y; c.r1 = b.x; c.i1 = b.y;
}
__device__ __forceinline__ void acc_store(const CAcc& c, double2* tl, int lane) {
    const int r = lane >> 2, c0 = 2 * (lane & 3);
    tl[sw(r, c0)] = make_double2(c.r0, c.i0);
    tl[sw(r, c0 + 1)] = make_double2(c.r1, c.i1);
}

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// ---- TMA / mbarrier (S1)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_tile(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

}  // namespace dm

// tmA: 3-D tensor map over A viewed as doubles {2n (re/im of a row), n rows, batch}, box
// {16, 8, 1} (one 8 x 8 complex tile), 128-byte swizzle.  X: any layout (element (i, j) of
// matrix b at X[b*sXm + (i*n + j)*sXe]); info[b] as for every kernel.
__global__ void __launch_bounds__(dm::NT, 5)
k_dmma(const __grid_constant__ CUtensorMap tmA, int64_t batch, double2* X, int64_t sXm, int64_t sXe,
       int32_t* __restrict__ info)
{
    using namespace dm;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    double2* Tl = reinterpret_cast<double2*>(sm);                       // tile p at Tl + 64 p
    double2* Vb = reinterpret_cast<double2*>(sm + OFF_V);               // warp w's V at Vb + 64 w
    double* invs = reinterpret_cast<double*>(sm + OFF_INV);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
    int* s_inf = reinterpret_cast<int*>(sm + OFF_BAR + 8);
#define TILE(I, J) (Tl + 64 * tidx((I), (J)))

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane >> 2, q = lane & 3;             // accumulator row, column pair
    const int64_t b = blockIdx.x;

    // ------------------------------------------------------------ S1: the 36 upper tiles
    if (tid == 0) {
        mbar_init(bar, 1);
        *s_inf = 0;
    }
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(bar, NTILE * TILE_B);
        for (int I = 0; I < NTL; I++)
            for (int J = I; J < NTL; J++) tma_load_tile(TILE(I, J), &tmA, 16 * J, 8 * I, int(b), bar);
    }
    mbar_wait(bar, 0);

    // ============================================================== factorisation, panels up
#pragma unroll 1
    for (int K = 0; K < NTL; K++) {
        if (warp == 0) {
            // ---- F1 on the diagonal tile, then F2a in registers
            CAcc a;
            acc_load(a, TILE(K, K), lane);
#pragma unroll 1
            for (int P = 0; P < K; P++) {
#pragma unroll
                for (int s = 0; s < 2; s++) {
                    const double2 u = fb(TILE(P, K), lane, s);        // A = -conj(R_PK)^T
                    const double2 v = fb(TILE(P, K), lane, s);        // B = R_PK
                    cmma(a, negd(u.x), u.y, negd(u.y), v.x, v.y);
                }
            }
            int inf = 0;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const double t = shfl_d((i & 1) ? a.r1 : a.r0, i * 4 + (i >> 1));   // Re a'_ii
                const bool bad = !(t > 0.0);
                if (bad && inf == 0) inf = K * 8 + i + 1;
                const double iv = rsqrt_fast(bad ? 1.0 : t);                        // 1 / r_ii
                if (r == i) { a.r0 *= iv; a.i0 *= iv; a.r1 *= iv; a.i1 *= iv; }    // row i of R (eq. 4)
                if (lane == 0) invs[K * 8 + i] = iv;
                if (i < 7) {
                    const int sj = i * 4 + q, sm_ = i * 4 + (r >> 1);
                    const double br0 = shfl_d(a.r0, sj), bi0 = shfl_d(a.i0, sj);    // r_ij, my columns
                    const double br1 = shfl_d(a.r1, sj), bi1 = shfl_d(a.i1, sj);
                    const double x0 = shfl_d(a.r0, sm_), y0 = shfl_d(a.i0, sm_);    // r_i,r (my row)
                    const double x1 = shfl_d(a.r1, sm_), y1 = shfl_d(a.i1, sm_);
                    const double ur = (r & 1) ? x1 : x0, ui = (r & 1) ? y1 : y0;
                    if (r > i) {                                                      // a'_rj -= conj(r_ir) r_ij
                        a.r0 = fma(-ur, br0, a.r0); a.r0 = fma(-ui, bi0, a.r0);
                        a.i0 = fma(-ur, bi0, a.i0); a.i0 = fma(ui, br0, a.i0);
                        a.r1 = fma(-ur, br1, a.r1); a.r1 = fma(-ui, bi1, a.r1);
                        a.i1 = fma(-ur, bi1, a.i1); a.i1 = fma(ui, br1, a.i1);
                    }
                }
            }
            acc_store(a, TILE(K, K), lane);
            if (lane == 0 && inf && *s_inf == 0) *s_inf = inf;
            __syncthreads();
            __syncthreads();
        } else {
            // ---- F1 on the off-diagonal tiles J = K+1+u, u = warp-1, warp+2, warp+5
            const int nt = (NTL - 1 - K - (warp - 1) + 2) / 3 > 0 ? (NTL - 1 - K - (warp - 1) + 2) / 3 : 0;
            CAcc a[3];
#pragma unroll
            for (int c = 0; c < 3; c++)
                if (c < nt) acc_load(a[c], TILE(K, K + warp + 3 * c), lane);
#pragma unroll 1
            for (int P = 0; P < K; P++) {
#pragma unroll
                for (int s = 0; s < 2; s++) {
                    const double2 u = fb(TILE(P, K), lane, s);
                    const double ar = negd(u.x), ai = u.y, nai = negd(u.y);
#pragma unroll
                    for (int c = 0; c < 3; c++) {
                        if (c < nt) {
                            const double2 v = fb(TILE(P, K + warp + 3 * c), lane, s);
                            cmma(a[c], ar, ai, nai, v.x, v.y);
                        }
                    }
                }
            }
            __syncthreads();                           // R_KK and 1/r_kk are in shared memory
            // ---- F2b: forward substitution through R_KK^H (eq. 4) on the accumulators
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const double iv = invs[K * 8 + i];
                const double2 u = TILE(K, K)[sw(i, r)];                // r_i,r (upper for r > i)
                const int sj = i * 4 + q;
#pragma unroll
                for (int c = 0; c < 3; c++) {
                    if (c < nt) {
                        CAcc& x = a[c];
                        if (r == i) { x.r0 *= iv; x.i0 *= iv; x.r1 *= iv; x.i1 *= iv; }
                        const double br0 = shfl_d(x.r0, sj), bi0 = shfl_d(x.i0, sj);
                        const double br1 = shfl_d(x.r1, sj), bi1 = shfl_d(x.i1, sj);
                        if (r > i) {
                            x.r0 = fma(-u.x, br0, x.r0); x.r0 = fma(-u.y, bi0, x.r0);
                            x.i0 = fma(-u.x, bi0, x.i0); x.i0 = fma(u.y, br0, x.i0);
                            x.r1 = fma(-u.x, br1, x.r1); x.r1 = fma(-u.y, bi1, x.r1);
                            x.i1 = fma(-u.x, bi1, x.i1); x.i1 = fma(u.y, br1, x.i1);
                        }
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < 3; c++)
                if (c < nt) acc_store(a[c], TILE(K, K + warp + 3 * c), lane);
            __syncthreads();
        }
    }
    __syncthreads();
    const int inf = *s_inf;

    if (inf == 0) {
    // ============================================================== inversion, panels down
#pragma unroll 1
    for (int K = NTL - 1; K >= 0; K--) {
        // ---- I1: C_KJ for the tiles J = K+1+warp, K+5+warp
        const int nt = (NTL - 1 - K - warp + 3) / 4 > 0 ? (NTL - 1 - K - warp + 3) / 4 : 0;
        CAcc a[2];
        czero(a[0]);
        czero(a[1]);
#pragma unroll 1
        for (int M = K + 1; M < NTL; M++) {
#pragma unroll
            for (int s = 0; s < 2; s++) {
                const double2 u = fa(TILE(K, M), lane, s);            // A = R_KM
                const double nui = negd(u.y);
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    if (c < nt) {
                        const int J = K + 1 + warp + 4 * c;
                        double2 v;
                        if (M <= J) v = fb(TILE(M, J), lane, s);                       // X_MJ
                        else { v = fa(TILE(J, M), lane, s); v.y = negd(v.y); }          // conj(X_JM)^T
                        cmma(a[c], u.x, u.y, nui, v.x, v.y);
                    }
                }
            }
        }
        // ---- I2: back substitution through R_KK (eqs. 22-24): rows k = 7..0 of the tile
#pragma unroll
        for (int k = 7; k >= 0; k--) {
            const double niv = -invs[K * 8 + k];
            const double2 u = TILE(K, K)[sw(r, k)];                   // r_rk (upper for r < k)
            const int sj = k * 4 + q;
#pragma unroll
            for (int c = 0; c < 2; c++) {
                if (c < nt) {
                    CAcc& x = a[c];
                    if (r == k) { x.r0 *= niv; x.i0 *= niv; x.r1 *= niv; x.i1 *= niv; }   // x_kj
                    if (k > 0) {
                        const double br0 = shfl_d(x.r0, sj), bi0 = shfl_d(x.i0, sj);
                        const double br1 = shfl_d(x.r1, sj), bi1 = shfl_d(x.i1, sj);
                        if (r < k) {                                      // c_rj += r_rk x_kj
                            x.r0 = fma(u.x, br0, x.r0); x.r0 = fma(-u.y, bi0, x.r0);
                            x.i0 = fma(u.x, bi0, x.i0); x.i0 = fma(u.y, br0, x.i0);
                            x.r1 = fma(u.x, br1, x.r1); x.r1 = fma(-u.y, bi1, x.r1);
                            x.i1 = fma(u.x, bi1, x.i1); x.i1 = fma(u.y, br1, x.i1);
                        }
                    }
                }
            }
        }
        // ---- I3: V_w = sum over this warp's tiles of R_KJ X_KJ^H (B = X^H from the registers)
        {
            CAcc v;
            czero(v);
#pragma unroll
            for (int c = 0; c < 2; c++) {
                if (c < nt) {
                    const int J = K + 1 + warp + 4 * c;
#pragma unroll
                    for (int s = 0; s < 2; s++) {
                        const double2 u = fa(TILE(K, J), lane, s);     // R_KJ
                        const double xr = s ? a[c].r1 : a[c].r0, xi = s ? a[c].i1 : a[c].i0;
                        cmma(v, u.x, u.y, negd(u.y), xr, negd(xi));
                    }
                }
            }
            acc_store(v, Vb + 64 * warp, lane);
        }
        __syncthreads();                               // every R_KT read is done
#pragma unroll
        for (int c = 0; c < 2; c++)
            if (c < nt) acc_store(a[c], TILE(K, K + 1 + warp + 4 * c), lane);
        // ---- I4: the diagonal tile, warp 0, lane j < 8 owns column j of X_KK
        if (warp == 0) {
            const int j = lane & 7;
            double2 xc[8];
#pragma unroll
            for (int m = 0; m < 8; m++) xc[m] = make_double2(0.0, 0.0);
            const double2* Rkk = TILE(K, K);
#pragma unroll
            for (int k = 7; k >= 0; k--) {
                const double ik = invs[K * 8 + k];
                // x_kj, j > k: -(1/r_kk)(V_kj + sum_{m>k} r_km x~_mj)
                double2 sv = Vb[sw(k, j)];
#pragma unroll
                for (int w = 1; w < 4; w++) { const double2 p = Vb[64 * w + sw(k, j)]; sv.x += p.x; sv.y += p.y; }
#pragma unroll
                for (int m = 7; m > k; m--) {
                    const double2 rk = Rkk[sw(k, m)];
                    sv.x = fma(rk.x, xc[m].x, sv.x); sv.x = fma(-rk.y, xc[m].y, sv.x);
                    sv.y = fma(rk.x, xc[m].y, sv.y); sv.y = fma(rk.y, xc[m].x, sv.y);
                }
                if (j > k) xc[k] = make_double2(-ik * sv.x, -ik * sv.y);
                // the row goes to the diagonal lane k as the lower part of its column (mirror),
                // and lane k forms x_kk = (1/r_kk)(1/r_kk - Re(V_kk + sum_{m>k} r_km conj(x_km)))
                double p = Vb[sw(k, k)].x;
#pragma unroll
                for (int w = 1; w < 4; w++) p += Vb[64 * w + sw(k, k)].x;
#pragma unroll
                for (int m = 7; m > k; m--) {
                    const double gx = shfl_d(xc[k].x, m), gy = shfl_d(xc[k].y, m);   // x_km
                    if (j == k) {
                        const double2 rk = Rkk[sw(k, m)];
                        xc[m] = make_double2(gx, negd(gy));
                        p = fma(rk.x, gx, p);
                        p = fma(rk.y, gy, p);
                    }
                }
                if (j == k) xc[k] = make_double2(ik * (ik - p), 0.0);
            }
            __syncwarp();
            if (lane < 8) {
                double2* D = TILE(K, K);
#pragma unroll
                for (int m = 0; m < 8; m++) D[sw(m, j)] = xc[m];
            }
        }
        __syncthreads();
    }
    }

    // ------------------------------------------------------------------ S5: store X
    double2* Xb = X + b * sXm;
    const double nan = qnan<double>();
#pragma unroll 1
    for (int tt = warp; tt < NTL * NTL; tt += NT / 32) {
        const int I = tt >> 3, J = tt & 7;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int rr = (lane >> 3) + 4 * h, cc = lane & 7;
            double2 v;
            if (I <= J) v = TILE(I, J)[sw(rr, cc)];
            else { v = TILE(J, I)[sw(cc, rr)]; v.y = -v.y; }
            if (inf) v = make_double2(nan, nan);
            __stcs(Xb + int64_t((8 * I + rr) * N + 8 * J + cc) * sXe, v);
        }
    }
    if (tid == 0) info[b] = inf;
#undef TILE
}

}  // namespace hpdinv
