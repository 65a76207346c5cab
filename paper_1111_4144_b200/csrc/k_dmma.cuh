// k_dmma.cuh -- n = 64, complex128, Cholesky: ONE MATRIX PER WARP, shared-memory resident, the
// GEMM-shaped updates on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64) -- the config-4
// kernel.
//
// Why DMMA: on B200 the FP64 DMMA path reaches 37.05 TF/s (tools/mma_peaks.cu,
// profiles/r02_mma_peaks.txt) against 33.4 for DFMA, on the same FP64 datapath, and one DMMA
// instruction carries 256 FMAs instead of 32: the blocked algorithm stops being bound by
// instruction issue, shared-memory operand traffic and register-bank conflicts (the round-1
// k_blk ran 48k warp instructions per matrix for 16k DFMA).
// Why one matrix per warp: no block-level barrier anywhere -- the serial phases of one warp
// (pivots, the in-tile substitutions, the diagonal-tile inversion) overlap the DMMA phases of
// the other warps of the SM -- and 255 registers per thread (6 warps per SM, 216 KB of tiles).
// Persistent: warp w of CTA c inverts matrices c*6 + w, + 6*gridDim, ...; while it stores
// matrix b it already loads matrix b + 6*gridDim into the tiles it has stored (TMA, one
// mbarrier per tile row, so panel K of the next matrix waits only for tile row K).
//
// Storage (per warp, 36 KB): only the 36 UPPER 8 x 8 tiles (I <= J) of the working matrix,
// complex interleaved, 1 KB per tile; element (r, c) of a tile at 16-byte slot r*8 + (c ^ r)
// -- the 128-byte TMA swizzle, so S1 is 36 cp.async.bulk.tensor tile loads.  Every fragment
// access pattern below is bank-conflict free in this layout (quarter-warp phases of the
// 16-byte accesses), provided the k index of k-step s of the m8n8k4 MMA runs over the tile
// columns {s, 2+s, 4+s, 6+s}: lane t (q = t % 4) then holds k = 2q + s, exactly the column of
// its own accumulator element e = s -- so a conjugate-transposed operand X^H is fed to the next
// MMA straight from the accumulator registers (I3).  Tile (I, J) holds A -> R (the factor,
// upper) -> X (in place, App. A.1); the diagonal tile holds R_KK in its upper half, then the
// FULL Hermitian X_KK.
//
// Factor (eqs. 3-4), panels K = 0..7 (left-looking: the sums of eqs. 3-4 over k < 8K at once):
//   F1  A_KJ -= sum_{P<K} R_PK^H R_PJ  for J >= K       (DMMA, accumulators start at A_KJ)
//   F2a R_KK by the right-looking recursion of eqs. 3-4 on the accumulator registers (pivots
//       and rows broadcast by shuffles); info = first k with !(t_k > 0)
//   F2b R_KJ = R_KK^-H A_KJ, J > K: the forward substitution of eq. 4 on the accumulators
// Proposed inversion (eqs. 20-24), panels K = 7..0, T = K+1..7:
//   I1  C_KJ = sum_{M in T} R_KM X~_MJ  for J in T    (DMMA; X~_MJ = X_JM^H read transposed)
//   I2  x_kj = -(1/r_kk)(C_kj + sum_{m in K, m>k} r_km x_mj), k = 7..0 (registers, shuffles)
//   I3  V = sum_{J in T} R_KJ X_KJ^H                   (DMMA, X^H from the accumulators)
//   I4  X_KK by the recursion of eq. 23 with V_kj added (lane j owns column j; the row
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
constexpr int WPB = 6;                               // warps (matrices) per CTA, one CTA per SM
constexpr int NT = 32 * WPB;
constexpr int TILES_B = (NTILE + 1) * 1024;          // 36 tiles + 1 scratch tile per warp
constexpr int AUX_B = 64 * 8 + 8 * 8;                // per warp: 1/r_kk (64 doubles), 8 mbarriers
constexpr int SMEM = WPB * (TILES_B + AUX_B) + 1024; // + alignment slack (TMA 128B swizzle)

__host__ __device__ constexpr int tidx(int I, int J) { return I * NTL - I * (I - 1) / 2 + (J - I); }
// first slot of tile row I (tile (I, J) = rowbase(I) + 64 J, double2 units; J >= I only)
__device__ __forceinline__ int rowbase(int I) { return 64 * (7 * I - (I * (I - 1)) / 2); }
__host__ __device__ constexpr int sw(int r, int c) { return r * 8 + (c ^ r); }

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

// c += A B for one k-step: (ar, ai) the A fragment, nai = -ai, (br, bi) the B fragment
__device__ __forceinline__ void cmma(CAcc& c, double ar, double ai, double nai, double br, double bi) {
    dmma(c.r0, c.r1, ar, br);
    dmma(c.i0, c.i1, ar, bi);
    dmma(c.r0, c.r1, nai, bi);
    dmma(c.i0, c.i1, ai, br);
}

__device__ __forceinline__ void acc_load(CAcc& c, const double2* tl, int o0, int o1) {
    const double2 a = tl[o0], b = tl[o1];
    c.r0 = a.x; c.i0 = a.y; c.r1 = b.x; c.i1 = b.y;
}
__device__ __forceinline__ void acc_store(const CAcc& c, double2* tl, int o0, int o1) {
    tl[o0] = make_double2(c.r0, c.i0);
    tl[o1] = make_double2(c.r1, c.i1);
}

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// x_rj -= conj(u) * b for both accumulator elements (b0, b1 broadcast down the columns)
__device__ __forceinline__ void acc_fms_conj(CAcc& x, double2 u, double br0, double bi0, double br1, double bi1) {
    x.r0 = fma(-u.x, br0, x.r0); x.r0 = fma(-u.y, bi0, x.r0);
    x.i0 = fma(-u.x, bi0, x.i0); x.i0 = fma(u.y, br0, x.i0);
    x.r1 = fma(-u.x, br1, x.r1); x.r1 = fma(-u.y, bi1, x.r1);
    x.i1 = fma(-u.x, bi1, x.i1); x.i1 = fma(u.y, br1, x.i1);
}
// x_rj += u * b
__device__ __forceinline__ void acc_fma(CAcc& x, double2 u, double br0, double bi0, double br1, double bi1) {
    x.r0 = fma(u.x, br0, x.r0); x.r0 = fma(-u.y, bi0, x.r0);
    x.i0 = fma(u.x, bi0, x.i0); x.i0 = fma(u.y, br0, x.i0);
    x.r1 = fma(u.x, br1, x.r1); x.r1 = fma(-u.y, bi1, x.r1);
    x.i1 = fma(u.x, bi1, x.i1); x.i1 = fma(u.y, br1, x.i1);
}
__device__ __forceinline__ void acc_scale(CAcc& x, double s) { x.r0 *= s; x.i0 *= s; x.r1 *= s; x.i1 *= s; }

// ---- TMA / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
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
// tile row I of matrix b: arm its barrier and load tiles (I, I..7)
__device__ __forceinline__ void load_row(double2* Tw, const CUtensorMap* tm, int I, int64_t b, uint64_t* bar) {
    mbar_expect_tx(bar, unsigned(NTL - I) * 1024u);
    for (int J = I; J < NTL; J++) tma_load_tile(Tw + 64 * tidx(I, J), tm, 16 * J, 8 * I, int(b), bar);
}

}  // namespace dm

// tmA: 3-D tensor map over A viewed as doubles {2n (re/im of a row), n rows, batch}, box
// {16, 8, 1} (one 8 x 8 complex tile), 128-byte swizzle.  X: any layout (element (i, j) of
// matrix b at X[b*sXm + (i*n + j)*sXe]); info[b] as for every kernel.
__global__ void __launch_bounds__(dm::NT, 1)
k_dmma(const __grid_constant__ CUtensorMap tmA, int64_t batch, double2* X, int64_t sXm, int64_t sXe,
       int32_t* __restrict__ info)
{
    using namespace dm;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pad = int((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    double2* Tw = reinterpret_cast<double2*>(smem_raw + pad + warp * TILES_B);      // this warp's tiles
    double* invs = reinterpret_cast<double*>(smem_raw + pad + WPB * TILES_B + warp * AUX_B);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + pad + WPB * TILES_B + warp * AUX_B + 64 * 8);
    double2* Ws = Tw + 64 * NTILE;                                                  // scratch tile
#define TILE(I, J) (Tw + rowbase(I) + 64 * (J))

    const int r = lane >> 2, q = lane & 3;             // accumulator row, column pair
    // per-lane fragment slots: oa[s] = (r, 2q+s) (A as stored / accumulator element s),
    // ob[s] = (2q+s, r) (B as stored / A transposed)
    const int oa0 = sw(r, 2 * q), oa1 = sw(r, 2 * q + 1);
    const int ob0 = sw(2 * q, r), ob1 = sw(2 * q + 1, r);

    const int64_t stride = int64_t(gridDim.x) * WPB;
    int64_t b = int64_t(blockIdx.x) * WPB + warp;
    if (lane == 0) {
        for (int I = 0; I < NTL; I++) mbar_init(&bar[I], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (b < batch)
            for (int I = 0; I < NTL; I++) load_row(Tw, &tmA, I, b, &bar[I]);
    }
    __syncwarp();

#pragma unroll 1
    for (unsigned it = 0; b < batch; b += stride, it++) {
        const unsigned par = it & 1u;
        int inf = 0;
        // ========================================================== factorisation, panels up
#pragma unroll 1
        for (int K = 0; K < NTL; K++) {
            mbar_wait(&bar[K], par);                       // tile row K of A has landed
            double2* tKK = TILE(K, K);
            // ---- F1 on the diagonal tile: A_KK -= sum_{P<K} R_PK^H R_PK
            CAcc d;
            acc_load(d, tKK, oa0, oa1);
#pragma unroll 1
            for (int P = 0; P < K; P++) {
                const double2* tPK = TILE(P, K);
#pragma unroll
                for (int s = 0; s < 2; s++) {
                    const double2 u = tPK[s ? ob1 : ob0];                 // A = -conj(R_PK)^T, B = R_PK
                    cmma(d, negd(u.x), u.y, negd(u.y), u.x, u.y);
                }
            }
            // ---- F2a: R_KK by the right-looking recursion of eqs. 3-4 on the accumulators, and
            //      E = R_KK^-H (the same row operations applied to I), for the panel solves.
            //      Step i broadcasts the unscaled row i and the pivot together; every lane scales
            //      by 1/r_ii itself (the update uses conj(a_ir) a_ij / t_i = conj(r_ir) r_ij).
            CAcc e;
            e.r0 = (r == 2 * q) ? 1.0 : 0.0;
            e.r1 = (r == 2 * q + 1) ? 1.0 : 0.0;
            e.i0 = 0.0;
            e.i1 = 0.0;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const int sp = i * 4 + (i >> 1), sj = i * 4 + q, sr = i * 4 + (r >> 1);
                const double t = shfl_d((i & 1) ? d.r1 : d.r0, sp);                 // Re a'_ii
                const double ar0 = shfl_d(d.r0, sj), ai0 = shfl_d(d.i0, sj);        // a'_ij, my columns
                const double ar1 = shfl_d(d.r1, sj), ai1 = shfl_d(d.i1, sj);
                const double er0 = shfl_d(e.r0, sj), ei0 = shfl_d(e.i0, sj);        // E_ij, my columns
                const double er1 = shfl_d(e.r1, sj), ei1 = shfl_d(e.i1, sj);
                const double x0 = shfl_d(d.r0, sr), y0 = shfl_d(d.i0, sr);          // a'_i,r (my row)
                const double x1 = shfl_d(d.r1, sr), y1 = shfl_d(d.i1, sr);
                const bool bad = !(t > 0.0);
                if (bad && inf == 0) inf = K * 8 + i + 1;
                const double tt = bad ? 1.0 : t;
                const double iv = rsqrt_fast(tt);                                    // 1 / r_ii
                const double iv2 = iv * iv;
                if (lane == 0) invs[K * 8 + i] = iv;
                if (r == i) { acc_scale(d, iv); acc_scale(e, iv); }                  // row i of R, of E
                if (r > i) {                                                          // rows below: -= conj(r_ir) r_i.
                    const double2 w = make_double2(((r & 1) ? x1 : x0) * iv2, ((r & 1) ? y1 : y0) * iv2);
                    acc_fms_conj(d, w, ar0, ai0, ar1, ai1);
                    acc_fms_conj(e, w, er0, ei0, er1, ei1);
                }
            }
            // diagonal tile: R_KK in the strict upper half, E = R_KK^-H (lower, diagonal 1/r_kk)
            {
                const bool up0 = r < 2 * q, up1 = r < 2 * q + 1;
                tKK[oa0] = up0 ? make_double2(d.r0, d.i0) : make_double2(e.r0, e.i0);
                tKK[oa1] = up1 ? make_double2(d.r1, d.i1) : make_double2(e.r1, e.i1);
            }
            // ---- F1 + F2b per off-diagonal tile: R_KJ = E (A_KJ - sum_{P<K} R_PK^H R_PJ) (eq. 4)
#pragma unroll 1
            for (int J = K + 1; J < NTL; J++) {
                double2* tKJ = TILE(K, J);
                CAcc a;
                acc_load(a, tKJ, oa0, oa1);
#pragma unroll 1
                for (int P = 0; P < K; P++) {
                    const double2* tP = TILE(P, 0);
#pragma unroll
                    for (int s = 0; s < 2; s++) {
                        const int ob = s ? ob1 : ob0;
                        const double2 u = tP[64 * K + ob], v = tP[64 * J + ob];
                        cmma(a, negd(u.x), u.y, negd(u.y), v.x, v.y);
                    }
                }
                acc_store(a, tKJ, oa0, oa1);                                        // A'_KJ, read back as B
                __syncwarp();
                const double2 b0 = tKJ[ob0], b1 = tKJ[ob1];
                __syncwarp();
                CAcc x;
                czero(x);
                cmma(x, e.r0, e.i0, negd(e.i0), b0.x, b0.y);
                cmma(x, e.r1, e.i1, negd(e.i1), b1.x, b1.y);
                acc_store(x, tKJ, oa0, oa1);
            }
            __syncwarp();
        }

        if (inf == 0) {
        // ========================================================== inversion, panels down
#pragma unroll 1
        for (int K = NTL - 1; K >= 0; K--) {
            const double2* rowK = TILE(K, 0);
            const double2* tKK = rowK + 64 * K;
            CAcc a[8];
#pragma unroll
            for (int J = 1; J < NTL; J++) czero(a[J]);
            // ---- I1: C_KJ = sum_{M in T} R_KM X~_MJ (A = R_KM; B = X_MJ, or X_JM^H for M > J)
#pragma unroll 1
            for (int M = K + 1; M < NTL; M++) {
                const double2* rowM = TILE(M, 0);
#pragma unroll
                for (int s = 0; s < 2; s++) {
                    const double2 u = rowK[64 * M + (s ? oa1 : oa0)];
                    const double nui = negd(u.y);
#pragma unroll
                    for (int J = 1; J < NTL; J++) {
                        if (J > K) {
                            double2 v;
                            if (M <= J) v = rowM[64 * J + (s ? ob1 : ob0)];
                            else { v = TILE(J, 0)[64 * M + (s ? oa1 : oa0)]; v.y = negd(v.y); }
                            cmma(a[J], u.x, u.y, nui, v.x, v.y);
                        }
                    }
                }
            }
            // ---- I2 + I3 per tile: X_KJ = -R_KK^-1 C_KJ (eqs. 22-24 for the rows of the panel,
            //      R_KK^-1 = E^H from the diagonal tile's lower half), then V += R_KJ X_KJ^H and
            //      X_KJ replaces R_KJ (every R_KT read of I1 is done)
            double ra0, ia0, ra1, ia1;                                             // A = -R_KK^-1
            {
                const double2 w0 = tKK[ob0], w1 = tKK[ob1];                        // E(2q+s, r)
                const bool v0 = 2 * q >= r, v1 = 2 * q + 1 >= r;
                ra0 = v0 ? negd(w0.x) : 0.0; ia0 = v0 ? w0.y : 0.0;
                ra1 = v1 ? negd(w1.x) : 0.0; ia1 = v1 ? w1.y : 0.0;
            }
            CAcc v;
            czero(v);
#pragma unroll
            for (int J = 1; J < NTL; J++) {
                if (J > K) {
                    acc_store(a[J], Ws, oa0, oa1);                                 // C_KJ, read back as B
                    __syncwarp();
                    const double2 c0 = Ws[ob0], c1 = Ws[ob1];
                    __syncwarp();
                    CAcc x;
                    czero(x);
                    cmma(x, ra0, ia0, negd(ia0), c0.x, c0.y);
                    cmma(x, ra1, ia1, negd(ia1), c1.x, c1.y);
                    double2* tKJ = TILE(K, J);
                    const double2 u0 = tKJ[oa0], u1 = tKJ[oa1];                    // R_KJ
                    cmma(v, u0.x, u0.y, negd(u0.y), x.r0, negd(x.i0));
                    cmma(v, u1.x, u1.y, negd(u1.y), x.r1, negd(x.i1));
                    acc_store(x, tKJ, oa0, oa1);
                }
            }
            // ---- I4: the diagonal tile; lane j (mod 8) owns column j of X_KK
            {
                const int j = lane & 7;
                double2 vc[8], xc[8];
#pragma unroll
                for (int k = 0; k < 8; k++) {                                      // V_kj to lane j
                    const int src = k * 4 + (j >> 1);
                    const double v0 = shfl_d(v.r0, src), w0 = shfl_d(v.i0, src);
                    const double v1 = shfl_d(v.r1, src), w1 = shfl_d(v.i1, src);
                    vc[k] = (j & 1) ? make_double2(v1, w1) : make_double2(v0, w0);
                    xc[k] = make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int k = 7; k >= 0; k--) {
                    const double ik = invs[K * 8 + k];
                    // x_kj, j > k: -(1/r_kk)(V_kj + sum_{m>k} r_km x~_mj), two chains
                    double2 s0 = vc[k], s1 = make_double2(0.0, 0.0);
#pragma unroll
                    for (int m = 7; m > k; m--) {
                        const double2 rk = tKK[sw(k, m)];
                        double2& s = ((7 - m) & 1) ? s1 : s0;
                        s.x = fma(rk.x, xc[m].x, s.x); s.x = fma(-rk.y, xc[m].y, s.x);
                        s.y = fma(rk.x, xc[m].y, s.y); s.y = fma(rk.y, xc[m].x, s.y);
                    }
                    if (j > k) xc[k] = make_double2(-ik * (s0.x + s1.x), -ik * (s0.y + s1.y));
                    // the row goes to the diagonal lane k as the lower part of its column (the
                    // mirror), which forms x_kk = (1/r_kk)(1/r_kk - Re(V_kk + sum r_km conj(x_km)))
                    double p = vc[k].x, p2 = 0.0;
#pragma unroll
                    for (int m = 7; m > k; m--) {
                        const double gx = shfl_d(xc[k].x, m), gy = shfl_d(xc[k].y, m);   // x_km
                        if (j == k) {
                            const double2 rk = tKK[sw(k, m)];
                            xc[m] = make_double2(gx, negd(gy));
                            double& pp = ((7 - m) & 1) ? p2 : p;
                            pp = fma(rk.x, gx, pp);
                            pp = fma(rk.y, gy, pp);
                        }
                    }
                    if (j == k) xc[k] = make_double2(ik * (ik - (p + p2)), 0.0);
                }
                __syncwarp();
                if (lane < 8) {
                    double2* D = TILE(K, K);
#pragma unroll
                    for (int m = 0; m < 8; m++) D[sw(m, j)] = xc[m];
                }
            }
            __syncwarp();
        }
        }

        // ============================================ S5: store X, prefetch the next matrix
        const int64_t bn = b + stride;
        double2* Xb = X + b * sXm;
        const double nan = qnan<double>();
        const int rr = lane >> 3, cc = lane & 7;
#pragma unroll 1
        for (int I = 0; I < NTL; I++) {
#pragma unroll 1
            for (int J = I; J < NTL; J++) {
                const double2* tl = TILE(I, J);
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int ro = rr + 4 * h;
                    double2 v = tl[sw(ro, cc)];
                    double2 w = tl[sw(cc, ro)];                                     // (J, I) = conj^T
                    w.y = negd(w.y);
                    if (inf) { v = make_double2(nan, nan); w = v; }
                    __stcs(Xb + int64_t((8 * I + ro) * N + 8 * J + cc) * sXe, v);
                    if (I < J) __stcs(Xb + int64_t((8 * J + ro) * N + 8 * I + cc) * sXe, w);
                }
            }
            __syncwarp();
            if (lane == 0 && bn < batch) {                 // row I is free: load it for the next matrix
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                load_row(Tw, &tmA, I, bn, &bar[I]);
            }
        }
        if (lane == 0) info[b] = inf;
    }
#undef TILE
}

}  // namespace hpdinv
