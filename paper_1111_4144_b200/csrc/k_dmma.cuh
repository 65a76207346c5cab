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
// Persistent: CTA c inverts matrices c*6 + w + 6*gridDim*k (its warps take them from a shared
// counter, the first six statically); while a warp stores matrix b it already loads its next
// matrix into the tiles it has stored (TMA, one mbarrier per tile row, so panel K of the next
// matrix waits only for tile row K).
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
//   F2a R_KK by the right-looking recursion of eqs. 3-4 on the accumulator registers (rows and
//       pivots broadcast through the tile); the same row operations on I give E = R_KK^-H;
//       info = first k with !(t_k > 0)
//   F2b R_KJ = E A'_KJ, J > K  (DMMA; DESIGN reading R22: the panel solve as a product with the
//       inverted 8 x 8 diagonal block)
// Proposed inversion (eqs. 20-24), panels K = 7..0, T = K+1..7:
//   I1  C_KJ = sum_{M in T} R_KM X~_MJ  for J in T    (DMMA; X~_MJ = X_JM^H read transposed)
//   I2  X_KJ = -E^H C_KJ                                (DMMA, R22)
//   I3  V = sum_{J in T} R_KJ X_KJ^H                   (DMMA, X^H from the accumulators)
//   I4  X_KK by the recursion of eq. 23 with V_kj added (lane j owns column j; the mirror of
//       each row goes through the tile's lower half to the diagonal lane), x_kk real
// The complex products of F1, I1 and I2 take the three-multiplication form (C3, reading R24):
// 3 real MMAs per complex k-step instead of 4.
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
constexpr int TILES_B = NTILE * 1024;                // 36 tiles per warp
constexpr int AUX_B = 64 * 8 + 8 * 8 + 8 * 8;        // per warp: 1/r_kk (64 doubles), 8 mbarriers, 8 I4 partials
constexpr int SMEM = WPB * (TILES_B + AUX_B) + 16 + 1024; // + the CTA's matrix counter + alignment slack (TMA 128B swizzle)

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

// the two halves of cmma: every first half of a k-step's tiles is issued before any second
// half, so the dependent MMA pairs of one tile are a whole k-step apart
__device__ __forceinline__ void cmma_h1(CAcc& c, double ar, double br, double bi) {
    dmma(c.r0, c.r1, ar, br);
    dmma(c.i0, c.i1, ar, bi);
}
__device__ __forceinline__ void cmma_h2(CAcc& c, double ai, double nai, double br, double bi) {
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

// complex product-sum in the three-multiplication form (Gauss): for C += A B the accumulator
// keeps P1 = sum ar br, P2 = sum ai bi and P3 = sum (ar + ai)(br + bi) -- three real MMAs per
// k-step instead of four -- and Re C = P1 - P2, Im C = P3 - P1 - P2 at the end (reading R24)
struct C3 { double p0, p1, q0, q1, s0, s1; };          // P1, P2, P3 for accumulator elements 0, 1
__device__ __forceinline__ void c3zero(C3& c) { c.p0 = c.p1 = c.q0 = c.q1 = c.s0 = c.s1 = 0.0; }
__device__ __forceinline__ void c3from(C3& c, const CAcc& x) {     // start from C = x
    c.p0 = x.r0; c.p1 = x.r1; c.q0 = 0.0; c.q1 = 0.0; c.s0 = x.r0 + x.i0; c.s1 = x.r1 + x.i1;
}
__device__ __forceinline__ void c3mma(C3& c, double ar, double ai, double as, double br, double bi, double bs) {
    dmma(c.p0, c.p1, ar, br);
    dmma(c.q0, c.q1, ai, bi);
    dmma(c.s0, c.s1, as, bs);
}
__device__ __forceinline__ void c3add(C3& c, const C3& d) {
    c.p0 += d.p0; c.p1 += d.p1; c.q0 += d.q0; c.q1 += d.q1; c.s0 += d.s0; c.s1 += d.s1;
}
__device__ __forceinline__ CAcc c3val(const C3& c) {
    CAcc x;
    x.r0 = c.p0 - c.q0; x.r1 = c.p1 - c.q1;
    x.i0 = (c.s0 - c.p0) - c.q0; x.i1 = (c.s1 - c.p1) - c.q1;
    return x;
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
// tile (I, J) of matrix b from shared memory to X (the map's 128-byte swizzle undoes the slots)
__device__ __forceinline__ void tma_store_tile(const CUtensorMap* tm, const void* src, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
        ::"l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int PENDING>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(PENDING) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// tile row I of matrix b: arm its barrier and load tiles (I, I..7)
__device__ __forceinline__ void load_row(double2* Tw, const CUtensorMap* tm, int I, int64_t b, uint64_t* bar) {
    mbar_expect_tx(bar, unsigned(NTL - I) * 1024u);
    for (int J = I; J < NTL; J++) tma_load_tile(Tw + 64 * tidx(I, J), tm, 16 * J, 8 * I, int(b), bar);
}

#ifdef HPDINV_DMMA_PROF
__device__ unsigned long long g_prof[16];   // per-phase cycles of lane 0, summed over warps
#define DM_PHASE(id)                                  \
    do {                                              \
        if (lane == 0) {                              \
            const long long t_ = clock64();           \
            prof_[prof_cur_] += t_ - prof_t_;         \
            prof_t_ = t_;                             \
            prof_cur_ = (id);                         \
        }                                             \
    } while (0)
#else
#define DM_PHASE(id) do {} while (0)
#endif

}  // namespace dm

// ---- the GEMM-shaped part of a panel with every index compile-time (one instantiation per
// panel K): no branch between the MMAs of different tiles, immediate shared-memory offsets,
// and the fragment loads free to be hoisted above the MMAs they feed.  (Predicated-off MMAs
// measured to cost pipe time, and a runtime tile count puts a branch around every tile.)
struct DmLane { int oa0, oa1, ob0, ob1, r, q; };
using dm::CAcc;

// F1 of the off-diagonal tiles + F2b:  R_KJ = E (A_KJ - sum_{P<K} R_PK^H R_PJ), J = K+1..7;
// E (the accumulator layout of F2a) is the A operand of F2b straight from registers
template <int K>
__device__ __forceinline__ void dm_factor_off(double2* __restrict__ Tw, const DmLane& L, const CAcc& e) {
    using namespace dm;
    constexpr int NT_ = NTL - 1 - K;
    CAcc a[NT_ > 0 ? NT_ : 1];
    C3 a3[NT_ > 0 ? NT_ : 1];
#pragma unroll
    for (int u = 0; u < NT_; u++) {
        acc_load(a[u], Tw + 64 * tidx(K, K + 1 + u), L.oa0, L.oa1);
        c3from(a3[u], a[u]);
    }
    // k-steps (P, s) software-pipelined: the next step's fragments are loaded before this step's MMAs
    double2 w = Tw[64 * tidx(0, K) + L.ob0];
    double2 v[NT_ > 0 ? NT_ : 1];
#pragma unroll
    for (int u = 0; u < NT_; u++) v[u] = Tw[64 * tidx(0, K + 1 + u) + L.ob0];
#pragma unroll
    for (int st = 0; st < 2 * K; st++) {
        const int P = st >> 1;
        double2 wn = w, vn[NT_ > 0 ? NT_ : 1];
        if (st + 1 < 2 * K) {
            const int Pn = (st + 1) >> 1, obn = ((st + 1) & 1) ? L.ob1 : L.ob0;
            wn = Tw[64 * tidx(Pn, K) + obn];                                 // A = -conj(R_PK)^T
#pragma unroll
            for (int u = 0; u < NT_; u++) vn[u] = Tw[64 * tidx(Pn, K + 1 + u) + obn];   // B = R_PJ
        }
        const double ar = negd(w.x), ai = w.y, as = w.y - w.x;
#pragma unroll
        for (int u = 0; u < NT_; u++) c3mma(a3[u], ar, ai, as, v[u].x, v[u].y, v[u].x + v[u].y);
        (void)P;
        w = wn;
#pragma unroll
        for (int u = 0; u < NT_; u++) v[u] = vn[u];
    }
    // A' through its own tile, read back as the B operand of E A'
#pragma unroll
    for (int u = 0; u < NT_; u++) {
        a[u] = c3val(a3[u]);
        acc_store(a[u], Tw + 64 * tidx(K, K + 1 + u), L.oa0, L.oa1);
    }
    __syncwarp();
    double2 b0[NT_ > 0 ? NT_ : 1], b1[NT_ > 0 ? NT_ : 1];
#pragma unroll
    for (int u = 0; u < NT_; u++) {
        b0[u] = Tw[64 * tidx(K, K + 1 + u) + L.ob0];
        b1[u] = Tw[64 * tidx(K, K + 1 + u) + L.ob1];
    }
    __syncwarp();
    // (four-multiplication form here: the three-multiplication one measured slower on this
    //  latency-bound 2-k-step product, 19.8 vs 18.7 ms at cfg4)
    const double ne0 = negd(e.i0), ne1 = negd(e.i1);
#pragma unroll
    for (int u = 0; u < NT_; u++) {
        czero(a[u]);
        cmma(a[u], e.r0, e.i0, ne0, b0[u].x, b0[u].y);
        cmma(a[u], e.r1, e.i1, ne1, b1[u].x, b1[u].y);
        acc_store(a[u], Tw + 64 * tidx(K, K + 1 + u), L.oa0, L.oa1);
    }
}

// I1 + I2 + I3 of panel K < 7: C_KJ = sum_{M in T} R_KM X~_MJ (X~_MJ = X_JM^H for M > J),
// X_KJ = -R_KK^-1 C_KJ (R_KK^-1 = E^H: the diagonal tile's lower half read transposed),
// v = sum_J R_KJ X_KJ^H; C goes through its own tile to be read back as B, each lane keeping
// its R_KJ fragments (its own slots) for I3
template <int K>
__device__ __forceinline__ void dm_invert_off(double2* Tw, const DmLane& L, CAcc& v) {
    using namespace dm;
    constexpr int NT_ = NTL - 1 - K;
    constexpr int M0 = K + 1;
    CAcc a[NT_];
    C3 a3[NT_];
#pragma unroll
    for (int u = 0; u < NT_; u++) c3zero(a3[u]);
    // k-steps (m, s) software-pipelined: the next step's fragments are loaded before this step's MMAs
    auto ldx = [&](int m, int s, int u) -> double2 {
        double2 x;
        if (m <= u) x = Tw[64 * tidx(M0 + m, M0 + u) + (s ? L.ob1 : L.ob0)];
        else { x = Tw[64 * tidx(M0 + u, M0 + m) + (s ? L.oa1 : L.oa0)]; x.y = negd(x.y); }
        return x;
    };
    double2 w = Tw[64 * tidx(K, M0) + L.oa0];
    double2 x[NT_];
#pragma unroll
    for (int u = 0; u < NT_; u++) x[u] = ldx(0, 0, u);
#pragma unroll
    for (int st = 0; st < 2 * NT_; st++) {
        double2 wn = w, xn[NT_];
        if (st + 1 < 2 * NT_) {
            const int mn = (st + 1) >> 1, sn = (st + 1) & 1;
            wn = Tw[64 * tidx(K, M0 + mn) + (sn ? L.oa1 : L.oa0)];           // A = R_KM
#pragma unroll
            for (int u = 0; u < NT_; u++) xn[u] = ldx(mn, sn, u);
        }
        const double ws = w.x + w.y;
#pragma unroll
        for (int u = 0; u < NT_; u++) c3mma(a3[u], w.x, w.y, ws, x[u].x, x[u].y, x[u].x + x[u].y);
        w = wn;
#pragma unroll
        for (int u = 0; u < NT_; u++) x[u] = xn[u];
    }
#pragma unroll
    for (int u = 0; u < NT_; u++) a[u] = c3val(a3[u]);
    const double2* tKK = Tw + 64 * tidx(K, K);
    double ra0, ia0, ra1, ia1;                                          // A = -R_KK^-1
    {
        const double2 w0 = tKK[L.ob0], w1 = tKK[L.ob1];                 // E(2q+s, r)
        const bool v0 = 2 * L.q >= L.r, v1 = 2 * L.q + 1 >= L.r;
        ra0 = v0 ? negd(w0.x) : 0.0; ia0 = v0 ? w0.y : 0.0;
        ra1 = v1 ? negd(w1.x) : 0.0; ia1 = v1 ? w1.y : 0.0;
    }
    double2 u0[NT_], u1[NT_];
#pragma unroll
    for (int u = 0; u < NT_; u++) {
        double2* tKJ = Tw + 64 * tidx(K, K + 1 + u);
        u0[u] = tKJ[L.oa0];                                             // R_KJ (own slots)
        u1[u] = tKJ[L.oa1];
        acc_store(a[u], tKJ, L.oa0, L.oa1);                             // C_KJ
    }
    __syncwarp();
    // I2 in the three-multiplication form; I3 (B straight from I2's accumulators) in the four-
    // multiplication form, which measured faster there (shorter chain, fewer registers)
    CAcc v2;
    czero(v2);
    const double as0 = ra0 + ia0, as1 = ra1 + ia1;
#pragma unroll
    for (int u = 0; u < NT_; u++) {
        const double2* tKJ = Tw + 64 * tidx(K, K + 1 + u);
        const double2 b0 = tKJ[L.ob0], b1 = tKJ[L.ob1];
        c3zero(a3[u]);
        c3mma(a3[u], ra0, ia0, as0, b0.x, b0.y, b0.x + b0.y);
        c3mma(a3[u], ra1, ia1, as1, b1.x, b1.y, b1.x + b1.y);
        a[u] = c3val(a3[u]);                                            // X_KJ
        // V += R_KJ X_KJ^H: B = conj(X_KJ) straight from the accumulators
        CAcc& vv = (u & 1) ? v2 : v;
        cmma(vv, u0[u].x, u0[u].y, negd(u0[u].y), a[u].r0, negd(a[u].i0));
        cmma(vv, u1[u].x, u1[u].y, negd(u1[u].y), a[u].r1, negd(a[u].i1));
    }
    __syncwarp();                                                       // every B read is done
#pragma unroll
    for (int u = 0; u < NT_; u++) acc_store(a[u], Tw + 64 * tidx(K, K + 1 + u), L.oa0, L.oa1);
    if (NT_ > 1) { v.r0 += v2.r0; v.r1 += v2.r1; v.i0 += v2.i0; v.i1 += v2.i1; }
}

// tmA: 3-D tensor map over A viewed as doubles {2n (re/im of a row), n rows, batch}, box
// {16, 8, 1} (one 8 x 8 complex tile), 128-byte swizzle.  X: any layout (element (i, j) of
// matrix b at X[b*sXm + (i*n + j)*sXe]); info[b] as for every kernel.
__global__ void __launch_bounds__(dm::NT, 1)
k_dmma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX, int xtma,
       int64_t batch, double2* X, int64_t sXm, int64_t sXe, int32_t* __restrict__ info)
{
    using namespace dm;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pad = int((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    double2* Tw = reinterpret_cast<double2*>(smem_raw + pad + warp * TILES_B);      // this warp's tiles
    double* invs = reinterpret_cast<double*>(smem_raw + pad + WPB * TILES_B + warp * AUX_B);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + pad + WPB * TILES_B + warp * AUX_B + 64 * 8);
    double* tpart = reinterpret_cast<double*>(smem_raw + pad + WPB * TILES_B + warp * AUX_B + 64 * 8 + 8 * 8);
#define TILE(I, J) (Tw + rowbase(I) + 64 * (J))

    const int r = lane >> 2, q = lane & 3;             // accumulator row, column pair
    // per-lane fragment slots: oa[s] = (r, 2q+s) (A as stored / accumulator element s),
    // ob[s] = (2q+s, r) (B as stored / A transposed)
    const int oa0 = sw(r, 2 * q), oa1 = sw(r, 2 * q + 1);
    const int ob0 = sw(2 * q, r), ob1 = sw(2 * q + 1, r);
    const DmLane L{oa0, oa1, ob0, ob1, r, q};

    // The CTA's j-th matrix is m(j) = (j / WPB) * stride + blockIdx.x * WPB + j % WPB; its warps take
    // j from a shared-memory counter (the first WPB statically), so the warps that have an SM
    // sub-partition to themselves (6 warps on 4) invert more matrices than the paired ones.
    const int64_t stride = int64_t(gridDim.x) * WPB;
    int* jnext = reinterpret_cast<int*>(smem_raw + pad + WPB * (TILES_B + AUX_B));
    if (threadIdx.x == 0) *jnext = WPB;
    __syncthreads();
    int64_t b = int64_t(blockIdx.x) * WPB + warp;
#ifdef HPDINV_DMMA_PROF
    long long prof_[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};   // wait F1d F2a F2b I1 I23 I4 S5 - -
    long long prof_t_ = clock64();
    int prof_cur_ = 8;
#endif
    if (lane == 0) {
        for (int I = 0; I < NTL; I++) mbar_init(&bar[I], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (b < batch)
            for (int I = 0; I < NTL; I++) load_row(Tw, &tmA, I, b, &bar[I]);
    }
    __syncwarp();

#pragma unroll 1
    for (unsigned it = 0; b < batch; it++) {
        const unsigned par = it & 1u;
        int inf = 0;
        // ========================================================== factorisation, panels up
#pragma unroll 1
        for (int K = 0; K < NTL; K++) {
            DM_PHASE(0);
            mbar_wait(&bar[K], par);                       // tile row K of A has landed
            DM_PHASE(1);
            double2* tKK = TILE(K, K);
            // ---- F1 on the diagonal tile: A_KK -= sum_{P<K} R_PK^H R_PK
            // four accumulators (P even / odd x k-step s) and split MMA halves: the dependent MMA
            // chain of the diagonal tile is a quarter as long
            CAcc d;
            acc_load(d, tKK, oa0, oa1);
            C3 d0, d1, d2, d3;
            c3from(d0, d);
            c3zero(d1);
            c3zero(d2);
            c3zero(d3);
            {
                // A = -conj(R_PK)^T = (-x, y), B = R_PK = (x, y): (ar + ai)(br + bi) = y^2 - x^2
                int P = 0;
#pragma unroll 1
                for (; P + 1 < K; P += 2) {
                    const double2 u0 = TILE(P, K)[ob0], u1 = TILE(P, K)[ob1];
                    const double2 w0 = TILE(P + 1, K)[ob0], w1 = TILE(P + 1, K)[ob1];
                    c3mma(d0, negd(u0.x), u0.y, u0.y - u0.x, u0.x, u0.y, u0.x + u0.y);
                    c3mma(d1, negd(u1.x), u1.y, u1.y - u1.x, u1.x, u1.y, u1.x + u1.y);
                    c3mma(d2, negd(w0.x), w0.y, w0.y - w0.x, w0.x, w0.y, w0.x + w0.y);
                    c3mma(d3, negd(w1.x), w1.y, w1.y - w1.x, w1.x, w1.y, w1.x + w1.y);
                }
                if (P < K) {
                    const double2 u0 = TILE(P, K)[ob0], u1 = TILE(P, K)[ob1];
                    c3mma(d0, negd(u0.x), u0.y, u0.y - u0.x, u0.x, u0.y, u0.x + u0.y);
                    c3mma(d1, negd(u1.x), u1.y, u1.y - u1.x, u1.x, u1.y, u1.x + u1.y);
                }
            }
            c3add(d1, d2);
            c3add(d1, d3);
            c3add(d0, d1);
            d = c3val(d0);
            DM_PHASE(2);
            // ---- F2a: R_KK by the right-looking recursion of eqs. 3-4 on the accumulators, and
            //      E = R_KK^-H (the same row operations applied to I), for the panel solves.
            //      Step i broadcasts the unscaled rows i of A' and of E through the diagonal tile
            //      (scratch until F2a ends: A' row i in tile row i, E row i in tile row i+4 mod 8,
            //      so consecutive steps never touch the same row); every lane scales by 1/r_ii
            //      itself (the update uses conj(a_ir) a_ij / t_i = conj(r_ir) r_ij).
            CAcc e;
            e.r0 = (r == 2 * q) ? 1.0 : 0.0;
            e.r1 = (r == 2 * q + 1) ? 1.0 : 0.0;
            e.i0 = 0.0;
            e.i1 = 0.0;
            __syncwarp();                                   // every F1d read of the tile is done
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const int ie = (i + 4) & 7;
                if (r == i) {
                    tKK[oa0] = make_double2(d.r0, d.i0);
                    tKK[oa1] = make_double2(d.r1, d.i1);
                    tKK[sw(ie, 2 * q)] = make_double2(e.r0, e.i0);
                    tKK[sw(ie, 2 * q + 1)] = make_double2(e.r1, e.i1);
                }
                __syncwarp();
                const double t = tKK[sw(i, i)].x;                                    // Re a'_ii
                const double2 a0 = tKK[sw(i, 2 * q)], a1 = tKK[sw(i, 2 * q + 1)];   // a'_ij, my columns
                const double2 e0 = tKK[sw(ie, 2 * q)], e1 = tKK[sw(ie, 2 * q + 1)]; // E_ij, my columns
                const double2 ar = tKK[sw(i, r)];                                    // a'_i,r (my row)
                const bool bad = !(t > 0.0);
                if (bad && inf == 0) inf = K * 8 + i + 1;
                const double tt = bad ? 1.0 : t;
                const double iv = rsqrt_fast(tt);                                    // 1 / r_ii
                const double iv2 = iv * iv;
                if (lane == 0) invs[K * 8 + i] = iv;
                if (r == i) { acc_scale(d, iv); acc_scale(e, iv); }                  // row i of R, of E
                if (r > i) {                                                          // rows below: -= conj(r_ir) r_i.
                    const double2 w = make_double2(ar.x * iv2, ar.y * iv2);
                    acc_fms_conj(d, w, a0.x, a0.y, a1.x, a1.y);
                    acc_fms_conj(e, w, e0.x, e0.y, e1.x, e1.y);
                }
            }
            __syncwarp();
            // diagonal tile: R_KK in the strict upper half, E = R_KK^-H (lower, diagonal 1/r_kk)
            {
                const bool up0 = r < 2 * q, up1 = r < 2 * q + 1;
                tKK[oa0] = up0 ? make_double2(d.r0, d.i0) : make_double2(e.r0, e.i0);
                tKK[oa1] = up1 ? make_double2(d.r1, d.i1) : make_double2(e.r1, e.i1);
            }
            DM_PHASE(3);
            // ---- F1 + F2b of the off-diagonal tiles: R_KJ = E (A_KJ - sum_{P<K} R_PK^H R_PJ) (eq. 4)
            switch (K) {
                case 0: dm_factor_off<0>(Tw, L, e); break;
                case 1: dm_factor_off<1>(Tw, L, e); break;
                case 2: dm_factor_off<2>(Tw, L, e); break;
                case 3: dm_factor_off<3>(Tw, L, e); break;
                case 4: dm_factor_off<4>(Tw, L, e); break;
                case 5: dm_factor_off<5>(Tw, L, e); break;
                case 6: dm_factor_off<6>(Tw, L, e); break;
                default: break;
            }
            __syncwarp();
        }

        if (inf == 0) {
        // ========================================================== inversion, panels down
#pragma unroll 1
        for (int K = NTL - 1; K >= 0; K--) {
            const double2* tKK = TILE(K, K);
            CAcc v;
            czero(v);
            DM_PHASE(4);
            // ---- I1 + I2 + I3 (v = V of the panel)
            switch (K) {
                case 0: dm_invert_off<0>(Tw, L, v); break;
                case 1: dm_invert_off<1>(Tw, L, v); break;
                case 2: dm_invert_off<2>(Tw, L, v); break;
                case 3: dm_invert_off<3>(Tw, L, v); break;
                case 4: dm_invert_off<4>(Tw, L, v); break;
                case 5: dm_invert_off<5>(Tw, L, v); break;
                case 6: dm_invert_off<6>(Tw, L, v); break;
                default: break;
            }
            DM_PHASE(5);
            DM_PHASE(6);
            // ---- I4: the diagonal tile by the recursion of eq. 23 with V added; lane j (mod 8) owns
            //      column j.  The lower half of the tile (E, dead after I2) carries V transposed
            //      (V_kj at slot (j, k)) and then, row by row, the mirror conj(x_kj) at slot (j, k),
            //      which the diagonal lane k reads back as the lower part of its column.
            {
                double2* D = TILE(K, K);
                if (r <= 2 * q) D[sw(2 * q, r)] = make_double2(v.r0, v.i0);
                if (r <= 2 * q + 1) D[sw(2 * q + 1, r)] = make_double2(v.r1, v.i1);
                __syncwarp();
                const int j = lane & 7;
                double2 xc[8], rkc[8], rkn[8];
#pragma unroll
                for (int m = 0; m < 8; m++) xc[m] = rkc[m] = rkn[m] = make_double2(0.0, 0.0);
                double2 vn = D[sw(j, 7)];
#ifndef HPDINV_DMMA_I4_CHAIN
                double2 rjn = D[sw(7, j)];                  // r_kj of the next step (upper half: R_KK)
#endif
#pragma unroll
                for (int k = 7; k >= 0; k--) {
                    const double ik = invs[K * 8 + k];
                    // x_kj, j > k: -(1/r_kk)(V_kj + sum_{m>k} r_km x~_mj), two chains.  Row k of
                    // R_KK and V_kj were loaded during step k+1 (neither changes in I4; slot
                    // (j, k) is overwritten by the mirror only in this step)
                    double2 s0 = vn, s1 = make_double2(0.0, 0.0);
#pragma unroll
                    for (int m = 7; m > k; m--) rkc[m] = rkn[m];
#ifndef HPDINV_DMMA_I4_CHAIN
                    const double2 rj = rjn;                 // r_kj (used by lanes j > k)
                    if (k > 0) rjn = D[sw(k - 1, j)];
#endif
                    if (k > 0) {
                        vn = D[sw(j, k - 1)];
#pragma unroll
                        for (int m = 7; m > k - 1; m--) rkn[m] = D[sw(k - 1, m)];
                    }
#pragma unroll
                    for (int m = 7; m > k; m--) {
                        const double2 rk = rkc[m];
                        double2& sa = ((7 - m) & 1) ? s1 : s0;
                        sa.x = fma(rk.x, xc[m].x, sa.x); sa.x = fma(-rk.y, xc[m].y, sa.x);
                        sa.y = fma(rk.x, xc[m].y, sa.y); sa.y = fma(rk.y, xc[m].x, sa.y);
                    }
#ifdef HPDINV_DMMA_I4_CHAIN
                    if (j > k) {
                        xc[k] = make_double2(-ik * (s0.x + s1.x), -ik * (s0.y + s1.y));
                        if (lane < 8) D[sw(j, k)] = make_double2(xc[k].x, negd(xc[k].y));   // the mirror
                    }
                    __syncwarp();
                    if (j == k) {
                        // x_kk = (1/r_kk)(1/r_kk - Re(V_kk + sum_{m>k} r_km conj(x_km)))
                        double p = D[sw(k, k)].x, p2 = 0.0;
#pragma unroll
                        for (int m = 7; m > k; m--) {
                            const double2 g = D[sw(m, k)];                          // conj(x_km)
                            const double2 rk = rkc[m];
                            xc[m] = g;
                            double& pp = ((7 - m) & 1) ? p2 : p;
                            pp = fma(rk.x, g.x, pp);
                            pp = fma(-rk.y, g.y, pp);
                        }
                        xc[k] = make_double2(ik * (ik - (p + p2)), 0.0);
                    }
#else
                    // lane j > k forms x_kj and its own term Re(r_kj conj(x_kj)) of the x_kk sum;
                    // the diagonal lane adds the terms pairwise (a tree of depth 3, not a chain)
                    if (j > k) {
                        xc[k] = make_double2(-ik * (s0.x + s1.x), -ik * (s0.y + s1.y));
                        const double t = fma(rj.x, xc[k].x, rj.y * xc[k].y);
                        if (lane < 8) {
                            D[sw(j, k)] = make_double2(xc[k].x, negd(xc[k].y));     // the mirror
                            tpart[j] = t;
                        }
                    }
                    __syncwarp();
                    if (j == k) {
                        // x_kk = (1/r_kk)(1/r_kk - Re(V_kk + sum_{m>k} r_km conj(x_km)))
                        double tt[8];
#pragma unroll
                        for (int m = 7; m > k; m--) {
                            xc[m] = D[sw(m, k)];                                    // conj(x_km)
                            tt[m] = tpart[m];
                        }
                        tt[k] = D[sw(k, k)].x;                                      // Re V_kk
#pragma unroll
                        for (int w = 1; w < 8; w *= 2)
#pragma unroll
                            for (int m = k; m + w <= 7; m += 2 * w) tt[m] += tt[m + w];
                        xc[k] = make_double2(ik * (ik - tt[k]), 0.0);
                    }
#endif
                }
                __syncwarp();
                if (lane < 8) {
#pragma unroll
                    for (int m = 0; m < 8; m++) D[sw(m, j)] = xc[m];
                }
            }
            __syncwarp();
        }
        }

        DM_PHASE(7);
        // ============================================ S5: store X, prefetch the next matrix
        int jn = 0;
        if (lane == 0) jn = atomicAdd(jnext, 1);
        jn = __shfl_sync(0xffffffffu, jn, 0);
        const int64_t bn = int64_t(jn / WPB) * stride + int64_t(blockIdx.x) * WPB + jn % WPB;
        double2* Xb = X + b * sXm;
        const double nan = qnan<double>();
        const int rr = lane >> 3, cc = lane & 7;
        if (xtma && !inf) {
            // X through the tensor map (contiguous X): the 36 upper tiles are bulk-stored by the
            // TMA engine straight from the swizzled tiles (one bulk group per tile row); the warp
            // writes only the 28 lower tiles, as conjugate transposes.  Tile row I is reloaded
            // for the next matrix once its group has been read out of shared memory.
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
#pragma unroll
                for (int I = 0; I < NTL; I++) {
#pragma unroll
                    for (int J = I; J < NTL; J++) tma_store_tile(&tmX, Tw + 64 * tidx(I, J), 16 * J, 8 * I, int(b));
                    bulk_commit();
                }
            }
            double2* Xl = Xb + (rr * N + cc);
#pragma unroll
            for (int I = 0; I < NTL; I++) {
#pragma unroll
                for (int J = I + 1; J < NTL; J++) {
                    const double2* tl = Tw + 64 * tidx(I, J);
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const int ro = rr + 4 * h;
                        double2 w = tl[sw(cc, ro)];                                 // (J, I) = conj^T
                        w.y = negd(w.y);
                        __stcs(Xl + ((8 * J + 4 * h) * N + 8 * I), w);
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    switch (I) {                                   // groups of rows > I may still be pending
                        case 0: bulk_wait_read<7>(); break;
                        case 1: bulk_wait_read<6>(); break;
                        case 2: bulk_wait_read<5>(); break;
                        case 3: bulk_wait_read<4>(); break;
                        case 4: bulk_wait_read<3>(); break;
                        case 5: bulk_wait_read<2>(); break;
                        case 6: bulk_wait_read<1>(); break;
                        default: bulk_wait_read<0>(); break;
                    }
                    if (bn < batch) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        load_row(Tw, &tmA, I, bn, &bar[I]);
                    }
                }
            }
        } else if (sXe == 1) {
            // contiguous X: every address is the lane base plus a compile-time offset
            double2* Xl = Xb + (rr * N + cc);
#pragma unroll
            for (int I = 0; I < NTL; I++) {
#pragma unroll
                for (int J = I; J < NTL; J++) {
                    const double2* tl = Tw + 64 * tidx(I, J);
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const int ro = rr + 4 * h;
                        double2 v = tl[sw(ro, cc)];
                        double2 w = tl[sw(cc, ro)];                                 // (J, I) = conj^T
                        w.y = negd(w.y);
                        if (inf) { v = make_double2(nan, nan); w = v; }
                        __stcs(Xl + ((8 * I + 4 * h) * N + 8 * J), v);
                        if (I < J) __stcs(Xl + ((8 * J + 4 * h) * N + 8 * I), w);
                    }
                }
                __syncwarp();
                if (lane == 0 && bn < batch) {             // row I is free: load it for the next matrix
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    load_row(Tw, &tmA, I, bn, &bar[I]);
                }
            }
        } else {
#pragma unroll 1
            for (int I = 0; I < NTL; I++) {
#pragma unroll 1
                for (int J = I; J < NTL; J++) {
                    const double2* tl = TILE(I, J);
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const int ro = rr + 4 * h;
                        double2 v = tl[sw(ro, cc)];
                        double2 w = tl[sw(cc, ro)];                                 // (J, I) = conj^T
                        w.y = negd(w.y);
                        if (inf) { v = make_double2(nan, nan); w = v; }
                        __stcs(Xb + int64_t((8 * I + ro) * N + 8 * J + cc) * sXe, v);
                        if (I < J) __stcs(Xb + int64_t((8 * J + ro) * N + 8 * I + cc) * sXe, w);
                    }
                }
                __syncwarp();
                if (lane == 0 && bn < batch) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    load_row(Tw, &tmA, I, bn, &bar[I]);
                }
            }
        }
        if (lane == 0) info[b] = inf;
        b = bn;
        DM_PHASE(8);
    }
    if (lane == 0) bulk_wait_all();                         // every bulk store of X has completed
#ifdef HPDINV_DMMA_PROF
    DM_PHASE(8);
    if (lane == 0)
        for (int i = 0; i < 10; i++) atomicAdd(&dm::g_prof[i], (unsigned long long)prof_[i]);
#endif
#undef TILE
}

}  // namespace hpdinv
