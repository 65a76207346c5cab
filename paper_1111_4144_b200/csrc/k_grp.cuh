// k_grp.cuh -- G lanes per matrix (G = 4 at n <= 16, 8 matrices per warp; G = 16 at n = 32, 2 per
// warp), every column held IN PLACE in registers: the config-3 kernel (n = 16, complex64,
// interleaved, 2^22 matrices) and the config-5 kernel (n = 32, complex64, LDL, contiguous).
//
// Design (why not one matrix per thread): the fully unrolled per-thread code of an n = 16
// matrix (~9.5k instructions, 150 KB) thrashes the instruction cache ("no_instruction" was the
// top stall at 6 warps/SM); splitting a matrix over G lanes divides the straight-line code per
// thread by G, and holding the columns in registers needs no shared-memory round trip per MAC.
//
// Lane q of a group owns the columns j = q + G*s (s = 0..C-1), dealt cyclically so all lanes
// have nearly the same active work at every step.  col[s][0..n-1] is column j of ONE working
// matrix that is, at every moment, R above the current row and X below it (App. A.1: row k of
// R is consumed by row k of X), so each lane holds n*C complex values and nothing else:
//   S1  load a_lj, l <= j (predicated: the strict lower part is never read);
//   S2  right-looking Cholesky (eqs. 3-4) / LDL (eqs. 10-11): at step i the owner of column i
//       forms the pivot t (info = first i with !(t > 0)), 1/r_ii (1/d_i) is broadcast by
//       shuffle, each lane scales its entries of row i and stores them in the group's packed
//       row store in shared memory; every lane then reads row i back (16-byte broadcast loads)
//       and updates a_lj -= conj(r_il) r_ij (LDL: conj(r_il) d_i r_ij), k = i ascending as in
//       the sums of eqs. 3-4;
//   S3  S = diag(1/r_ii) (eq. 24) / S~ = diag(1/d_i) (eq. 29): the reciprocals, kept in smem;
//   S4  rows k = n-1..0 (eqs. 22-24 / 27-29): R row k is read back from the row store; lane j
//       forms x_kj = -(1/r_kk) sum_{m>k} r_km x~_mj over its register column (x~_mj for m > k
//       is already X: the upper part computed in rows > k, the lower part gathered below);
//       each lane adds its columns' share of Re sum_{m>k} r_km conj(x_km) (r_kj is still in its
//       register column) and the G lanes combine it by shuffles; the new row goes, conjugated,
//       through a row buffer to the owner of column k, which takes it as the lower part of
//       column k (x_mk = conj(x_km), the mirror) and forms x_kk = (1/r_kk)(1/r_kk - Re sum) real
//       (measured: 8.5 -> 7.8 ms at config 5 against the owner forming the whole sum alone);
//   S5  every lane stores its columns (lower part: the bitwise conjugate written in S4).
// Dead storage is reused freely: a lane whose column j is not active at a step computes on
// entries of column j that are rewritten before they are read (lower part before its gather,
// rows <= j of a finished pivot), so the SIMT code needs no per-lane predicate except on the
// shared-memory stores.
#pragma once
#include "cplx.cuh"

namespace hpdinv {

template <typename T, int N, int G_>
struct GrpShape {
    static constexpr int G = G_;                      // lanes per matrix
    static constexpr int C = (N + G - 1) / G;         // columns per lane
    static constexpr int MPW = 32 / G;                // matrices per warp
#ifndef HPDINV_GRP_WARPS16
#define HPDINV_GRP_WARPS16 4
#endif
#ifndef HPDINV_GRP_WARPS32
#define HPDINV_GRP_WARPS32 8
#endif
    // n = 32: one 8-warp CTA per SM (248 registers) keeps the SM's warps in the same phase of
    // the 130 KB unrolled code (i-cache): 8.0 -> 7.5 ms at cfg5 against two 4-warp CTAs;
    // forcing lockstep with __syncthreads every 4/8/16 steps measured slower (8.1-8.5 ms)
    static constexpr int WARPS = N <= 16 ? HPDINV_GRP_WARPS16 : HPDINV_GRP_WARPS32;
    static constexpr int THREADS = 32 * WARPS;
    static constexpr int MPC = MPW * WARPS;           // matrices per CTA
    // n <= 16: 3 CTAs/SM caps ptxas at 170 registers (12 warps/SM); n = 32 (two 32-row columns
    // per lane) runs 8 warps/SM with up to 255 registers instead of spilling (measured faster)
#ifndef HPDINV_GRP_WSM16
#define HPDINV_GRP_WSM16 12   // resident warps per SM at n <= 16 (register budget)
#endif
    static constexpr int MIN_BLOCKS = N <= 16 ? (HPDINV_GRP_WSM16 / WARPS > 0 ? HPDINV_GRP_WSM16 / WARPS : 1)
                                              : (8 / WARPS > 0 ? 8 / WARPS : 1);
    static constexpr int P = sizeof(T) == 4 ? 2 : 1;  // complex elements per 16-byte load
    // packed row store: row i holds j = i..n-1 at offset roff(i) + (j - i), 16-byte aligned
    __host__ __device__ static constexpr int rlen(int i) { return ((N - i) + P - 1) / P * P; }
    __host__ __device__ static constexpr int roff(int i) { int o = 0; for (int k = 0; k < i; k++) o += rlen(k); return o; }
    static constexpr int RSZ = roff(N);
    static constexpr int ESZ = int(sizeof(cplx<T>));
    // per matrix: row store + X row buffer (n, padded) + reciprocals (n reals); the stride in
    // bytes is 16 mod 128 so the MPW groups of a warp hit distinct 16-byte bank quads
    static constexpr int RB = (N + P - 1) / P * P;     // one X row buffer (two, alternating)
    // COMPACT (n <= 16): 1/r_ii sits in the never-written diagonal slot of row i of the row
    // store, and the X row buffer of inversion step k is the dead row k+1 of the row store, so a
    // matrix needs the row store only: 3 CTAs fit the 132 KB carveout instead of 164 KB, L1 grows
    // 92 -> 124 KB, its sector hit rate 10.9 -> 21.5 % (the spills), cfg3 3.785 -> 3.735 ms
#ifndef HPDINV_GRP_NO_COMPACT
    static constexpr bool COMPACT = N <= 16;
#else
    static constexpr bool COMPACT = false;
#endif
    static constexpr int raw_full_bytes = (RSZ + 2 * RB) * ESZ + ((N * int(sizeof(T)) + 15) / 16) * 16;
    static constexpr int raw_bytes = COMPACT ? RSZ * ESZ : raw_full_bytes;
    static constexpr int MSTR_B = ((raw_bytes + 127) / 128) * 128 + 16;
    static constexpr size_t smem_bytes = size_t(MPC) * MSTR_B;
    // k_grp_solve keeps the separate row buffers and reciprocals
    static constexpr int MSTR_FULL_B = ((raw_full_bytes + 127) / 128) * 128 + 16;
    static constexpr size_t smem_bytes_full = size_t(MPC) * MSTR_FULL_B;
    // matrix -> row-store slot: with 8 groups per warp, group g sits at 16-byte bank quad
    // 2*(g%4) + g/4 (mod 8), so the 32-byte runs that the 4 groups of a half-warp write into
    // their row stores are disjoint (one wavefront per half-warp instead of two) while the 8
    // groups' 16-byte row broadcasts still hit 8 distinct quads
    __host__ __device__ static constexpr int slot(int mloc) {
        return MPW == 8 ? (mloc & ~7) + 2 * (mloc & 3) + ((mloc >> 2) & 1) : mloc;
    }
    // ---- staged global I/O (interleaved SoA, the CTA's MPC matrices contiguous in every plane):
    // one element plane of the CTA is a contiguous MPC*ESZ-byte segment in global memory, moved
    // by one cp.async.bulk; in shared memory the segments sit SPS bytes apart (= 32 mod 128): a
    // half-warp of 8-byte accesses is 4 matrices x the G = 4 consecutive planes of one warp
    // instruction, 4 disjoint 32-byte bank ranges, so a 256-byte LDS/STS is two wavefronts.  The staging area overlaps the row stores: the upper
    // planes of A before S2, then X (whole, or in two halves of rows) after S4.
    static constexpr int SPS = MPC * ESZ + 32;
    static constexpr int NUP = N * (N + 1) / 2;         // upper planes of A
    // X rows per store pass: two halves (the whole of X at once, 74 KB per CTA, leaves L1 almost
    // no capacity next to three CTAs' shared memory: cfg3 3.65 -> 4.49 ms)
    static constexpr int HROWS = (N + 1) / 2;
    __host__ __device__ static constexpr int pidx(int l, int j) { return l * N - l * (l - 1) / 2 + (j - l); }
    static constexpr size_t stage_bytes = size_t(NUP) * SPS > size_t(HROWS) * N * SPS ? size_t(NUP) * SPS
                                                                                        : size_t(HROWS) * N * SPS;
    static constexpr size_t region_bytes = stage_bytes > smem_bytes ? stage_bytes : smem_bytes;
    static constexpr size_t smem_bytes_staged = region_bytes + 16;   // + the mbarrier
};

namespace grp {
// X is streamed out and never re-read: evict-first stores (measured ~1 % faster at cfg3 and
// cfg5; evict-first LOADS cost 7 % at cfg5, where neighbouring lanes share AoS sectors in L1)
template <typename V>
__device__ __forceinline__ void st(V* p, V v) { __stcs(p, v); }
template <typename V>
__device__ __forceinline__ V ld(const V* p) { return __ldg(p); }
template <typename T>
__device__ __forceinline__ void lds_pair(const cplx<T>* p, int o, cplx<T>& e0, cplx<T>& e1) {
    if constexpr (sizeof(T) == 4) {
        const float4 v = *reinterpret_cast<const float4*>(p + (o & ~1));
        e0 = make_float2(v.x, v.y);
        e1 = make_float2(v.z, v.w);
    } else {
        e0 = p[o];
        e1 = e0;
    }
}
// bulk copies (async proxy: no LSU request, no L1 tag or data-stage wavefront per sector)
__device__ __forceinline__ uint32_t s32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(s32(dst)), "l"(src), "r"(bytes), "r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst), "r"(s32(src)), "r"(bytes) : "memory");
}
}  // namespace grp

// S1 + S2 of a lane group (shared by the inversion k_grp and the solve k_grp_solve): lane q
// loads the upper part of its columns j = q + G*s and runs the right-looking factorisation with
// the packed row store Rs; returns info.  See k_grp for the design notes.
template <typename T, int N, int GG, bool LDL, bool STG = false, bool CONTIG = false, bool INV_IN_ROW = false>
__device__ __forceinline__ int grp_factor(cplx<T> (&col)[GrpShape<T, N, GG>::C][N], const cplx<T>* __restrict__ Am,
                                          int64_t sAe, int q, cplx<T>* Rs, T* invs,
                                          const unsigned char* stq = nullptr) {
    using Sh = GrpShape<T, N, GG>;
    using V = cplx<T>;
    constexpr int G = Sh::G, C = Sh::C, P = Sh::P;
    constexpr unsigned FULL = 0xffffffffu;
    // ---------------------------------------------------------------- S1: load columns
    // (entries below the diagonal of a column are dead storage; Im a_jj is never read)
    if (STG && stq) {
        // from the staged upper planes: element (l, j = q + G*s) at stq + pidx(l, G*s) * SPS
        // (stq = staging base + this lane's matrix slot + q planes)
#pragma unroll
        for (int s = 0; s < C; s++) {
            const int j = q + G * s;
#pragma unroll
            for (int l = 0; l < N; l++) {
                col[s][l] = czero<T>();
                if (l <= G * s + G - 1 && l <= j && j < N)
                    col[s][l] = *reinterpret_cast<const V*>(stq + Sh::pidx(l, G * s) * Sh::SPS);
            }
        }
        __syncthreads();                                  // the staging area becomes row stores
    } else {
        // element (l, j = q + G*s): lane base + (l*n + G*s) * plane stride; the plane stride in
        // bytes is < 2^32 (checked by the launcher), so each address is one IMAD.WIDE
        // (CONTIG: sAe = 1, every address is the lane base plus a compile-time offset)
        const char* Ab = reinterpret_cast<const char*>(Am + q * (CONTIG ? 1 : sAe));
        const uint32_t seA = uint32_t(sAe * int64_t(sizeof(V)));
#pragma unroll
        for (int s = 0; s < C; s++) {
            const int j = q + G * s;
#pragma unroll
            for (int l = 0; l < N; l++) {
                col[s][l] = czero<T>();
                if (l <= G * s + G - 1 && l <= j && j < N)
                    col[s][l] = CONTIG ? grp::ld(reinterpret_cast<const V*>(Ab) + (l * N + G * s))
                                       : grp::ld(reinterpret_cast<const V*>(Ab + uint64_t(uint32_t(l * N + G * s)) * seA));
            }
        }
    }

    // -------------------------------------------------------- S2: right-looking factorisation
    int inf = 0;
#pragma unroll
    for (int i = 0; i < N; i++) {
        const int qi = i % G, si = i / G;
        // (taking the pivot from the owner's own diagonal update, as k_blk does, measured slower
        // here: 4.6 vs 4.1 ms at config 3 -- register pressure)
        const T t = (q == qi) ? col[si][i].x : T(1);    // non-owners feed 1: no slow paths
        const int bad0 = !(t > T(0));
        const T tt = bad0 ? T(1) : t;
        T iv;
        iv = LDL ? rcp_fast(tt) : rsqrt_fast(tt);      // short serial chain, exact at 1 (R9)
        iv = __shfl_sync(FULL, iv, qi, G);
        const int bad = __shfl_sync(FULL, bad0, qi, G);
        T di = T(0);
        if (LDL) di = __shfl_sync(FULL, tt, qi, G);
        if (bad && inf == 0) inf = i + 1;
        V* Ri = Rs + Sh::roff(i);
        if (q == 0) {
            if constexpr (INV_IN_ROW) reinterpret_cast<T*>(Ri)[0] = iv;   // COMPACT: Ri[0] is never a row entry
            else invs[i] = iv;
        }
        PMul<T> mul[C];
#pragma unroll
        for (int s = 0; s < C; s++) {
            if (G * s + G - 1 > i) {
                const int j = q + G * s;
                const V u = col[s][i];                   // a'_ij (unscaled)
                const V r = cscale(u, iv);               // r_ij (eq. 4 / eq. 11)
                col[s][i] = r;
                if (j > i && j < N) Ri[j - i] = r;
                // a'_lj -= conj(r_il) * r_ij (Cholesky) or conj(r_il) * d_i r_ij (LDL)
                const V w = LDL ? cscale(r, di) : r;
                mul[s] = pmul(mk<T>(-w.x, -w.y));
            }
        }
        __syncwarp();
#pragma unroll
        for (int o0 = 0; o0 < N; o0 += P) {
            if (o0 >= N - i) continue;
            V e[2];
            grp::lds_pair<T>(Ri, o0, e[0], e[1]);        // r_il, l = i + o0 + h
#pragma unroll
            for (int h = 0; h < P; h++) {
                const int oo = o0 + h;
                if (oo < 1 || oo >= N - i) continue;
                const int l = i + oo;
#pragma unroll
                for (int s = 0; s < C; s++) {
                    if (G * s + G - 1 >= l && G * s + G - 1 > i) {
                        PAcc<T> a = pacc(col[s][l]);
                        pmac_cb(a, mul[s], e[h]);
                        col[s][l] = pval(a);
                    }
                }
            }
        }
        // (no trailing __syncwarp: row i+1 of the row store is a different region, so the next
        //  step's pivot chain may overlap this step's update)
    }

    return inf;
}

// STG: staged global I/O (interleaved A and X, sAm = sXm = 1, even plane strides, 16-byte
// aligned bases -- checked by the launcher): a CTA holding MPC whole matrices moves its NUP
// upper planes of A and its n^2 planes of X as bulk copies of MPC*ESZ bytes each through the
// shared-memory staging area (GrpShape::SPS); a partial last CTA takes the per-lane path.
template <typename T, int N, int GG, bool LDL, bool STG = false, bool CONTIG = false>
__global__ void __launch_bounds__(GrpShape<T, N, GG>::THREADS, GrpShape<T, N, GG>::MIN_BLOCKS)
k_grp(int64_t batch, const cplx<T>* __restrict__ A, int64_t sAm, int64_t sAe,
      cplx<T>* X, int64_t sXm, int64_t sXe, int32_t* __restrict__ info)
{
    using Sh = GrpShape<T, N, GG>;
    using V = cplx<T>;
    constexpr int G = Sh::G, C = Sh::C, P = Sh::P;
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(16) unsigned char smem_raw[];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane & (G - 1), g = lane / G;
    const int mloc = warp * Sh::MPW + g;
    const int64_t b0 = int64_t(blockIdx.x) * Sh::MPC;
    int64_t b = b0 + mloc;
    const bool valid = b < batch;
    b = valid ? b : batch - 1;                        // the tail recomputes (never stores) the last matrix
    unsigned char* mbase = smem_raw + size_t(Sh::slot(mloc)) * Sh::MSTR_B;
    V* Rs = reinterpret_cast<V*>(mbase);                              // packed R rows
    V* rowbuf0 = Rs + Sh::RSZ;                                        // X row k (k odd: + RB)
    T* invs = Sh::COMPACT ? nullptr : reinterpret_cast<T*>(rowbuf0 + 2 * Sh::RB);   // 1/r_kk or 1/d_k

    // staged: the whole CTA is in the batch (uniform per CTA)
    const bool full = STG && b0 + Sh::MPC <= batch;
    const unsigned char* stq = nullptr;
#ifdef HPDINV_GRP_STAGE_LOADS
    if (STG && full) {
        uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + Sh::region_bytes);
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(grp::s32(bar)) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (warp == 0) {
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                             ::"r"(grp::s32(bar)), "r"(unsigned(Sh::NUP * Sh::MPC * Sh::ESZ)) : "memory");
            __syncwarp();
            for (int p = lane; p < Sh::NUP; p += 32) {
                int l = 0, r = p;
                while (r >= N - l) { r -= N - l; l++; }
                grp::bulk_g2s(smem_raw + p * Sh::SPS, A + b0 + int64_t(l * N + l + r) * sAe,
                              unsigned(Sh::MPC * Sh::ESZ), bar);
            }
        }
        asm volatile(
            "{\n.reg .pred p;\nWAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
            "@!p bra WAIT_%=;\n}\n" ::"r"(grp::s32(bar)) : "memory");
        stq = smem_raw + mloc * Sh::ESZ + q * Sh::SPS;
    }
#endif

    V col[C][N];
    int inf = grp_factor<T, N, GG, LDL, STG, CONTIG, Sh::COMPACT>(col, A + b * sAm, sAe, q, Rs, invs, stq);

    // ------------------------------------------------ S3/S4: proposed inversion, rows k = n..1
#pragma unroll
    for (int k = N - 1; k >= 0; k--) {
        const int qk = k % G, sk = k / G;
        // alternating: no reuse hazard between rows (COMPACT: row k+1 of the row store, dead
        // since every lane passed step k+1's __syncwarp after reading it; entry j at j - k - 1)
        V* rowbuf = Sh::COMPACT ? Rs + Sh::roff(k < N - 1 ? k + 1 : k) - (k + 1) : rowbuf0 + (k & 1) * Sh::RB;
        const V* Rk = Rs + Sh::roff(k);
        const T ik = Sh::COMPACT ? reinterpret_cast<const T*>(Rk)[0] : invs[k];
        V rk[N];                                        // r_km, m > k
#pragma unroll
        for (int o = 0; o < N; o += P) {
            if (o >= N - k) continue;
            V e0, e1;
            grp::lds_pair<T>(Rk, o, e0, e1);
            if (o >= 1) rk[k + o] = e0;
            if (P == 2 && o + 1 < N - k) rk[k + o + 1] = e1;
        }
        SAcc<T> acc[C];
#pragma unroll
        for (int s = 0; s < C; s++) sacc_zero(acc[s]);
#pragma unroll
        for (int m = 0; m < N; m++) {
            if (m <= k) continue;
#pragma unroll
            for (int s = 0; s < C; s++)
                if (G * s + G - 1 > k) smac(acc[s], rk[m], col[s][m]);
        }
        V xk[C];
        // x_kk: every lane forms its share of p = Re sum_{m>k} r_km conj(x_km) over its own
        // columns (r_kj is still in col[s][k], about to be overwritten by x_kj) and the G lanes
        // combine it by shuffles; the row goes to the row buffer already conjugated (the mirror)
        T pl = T(0);
#pragma unroll
        for (int s = 0; s < C; s++) {
            if (G * s + G - 1 > k) {
                const V a = sval(acc[s]);
                xk[s] = LDL ? mk<T>(-a.x, -a.y) : cscale(a, -ik);
                const V rkj = col[s][k];
                col[s][k] = xk[s];
                const int j = q + G * s;
                if (j > k && j < N) {
                    rowbuf[j] = conjz(xk[s]);
                    pl = re_dot_conj(pl, rkj, xk[s]);
                }
            }
        }
#pragma unroll
        for (int off = 1; off < G; off <<= 1) pl += __shfl_xor_sync(FULL, pl, off, G);
        __syncwarp();
        if (q == qk) {
            if constexpr (Sh::COMPACT) {
                // relative offsets: row k+1 of the row store is 16-byte aligned at entry k+1
#pragma unroll
                for (int o = 0; o < N; o += P) {
                    if (o >= N - k - 1) continue;
                    V e[2];
                    grp::lds_pair<T>(rowbuf + (k + 1), o, e[0], e[1]);
#pragma unroll
                    for (int h = 0; h < P; h++) {
                        const int m = k + 1 + o + h;
                        if (m < N) col[sk][m] = e[h];
                    }
                }
            } else {
#pragma unroll
            for (int o = 0; o < N; o += P) {
                if (o + P - 1 <= k) continue;
                V e[2];
                grp::lds_pair<T>(rowbuf, o, e[0], e[1]);
#pragma unroll
                for (int h = 0; h < P; h++) {
                    const int m = o + h;
                    if (m > k && m < N) col[sk][m] = e[h];
                }
            }
            }
            col[sk][k] = mk<T>(LDL ? ik - pl : ik * (ik - pl), T(0));
        }
    }

    // ------------------------------------------------------------------ S5: mirror + store
    if (STG && full) {
        // X through the staging area (whole, or in two halves of rows): every lane writes its columns
        // entries (m, j) of the half into plane m*n + j of its matrix slot, then each thread
        // bulk-stores planes of the half (MPC*ESZ bytes each, contiguous in X)
        __syncthreads();                                   // every row store / row buffer is dead
        unsigned char* stw = smem_raw + mloc * Sh::ESZ + q * Sh::SPS;
        const T nan = qnan<T>();
#pragma unroll
        for (int h = 0; h < (N + Sh::HROWS - 1) / Sh::HROWS; h++) {
            constexpr int H = Sh::HROWS;
            const int m0 = h * H;
#pragma unroll
            for (int s = 0; s < C; s++) {
                if (q + G * s < N) {
#pragma unroll
                    for (int m = 0; m < H; m++)
                        if (m0 + m < N)
                            *reinterpret_cast<V*>(stw + ((m * N) + G * s) * Sh::SPS) =
                                inf ? mk<T>(nan, nan) : col[s][m0 + m];
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            const int np = (N - m0 < H ? N - m0 : H) * N;
            for (int p = threadIdx.x; p < np; p += Sh::THREADS)
                grp::bulk_s2g(X + b0 + int64_t(m0 * N + p) * sXe, smem_raw + p * Sh::SPS,
                              unsigned(Sh::MPC * Sh::ESZ));
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            if (m0 + H < N) __syncthreads();               // the second half reuses the area
        }
        if (q == 0) info[b] = inf;
    } else if (valid) {
        // (storing each row as soon as it is final, inside S4, measured slower: 4.5 vs 4.1 ms cfg3)
        // every entry (m, j) is written once, by the owner of column j; a flagged matrix is
        // NaN-filled in the same store
        char* Xrow = reinterpret_cast<char*>(X + b * sXm + q * (CONTIG ? 1 : sXe));   // element (m, q + G s)
        const uint32_t seX = uint32_t(sXe * int64_t(sizeof(V)));
        const T nan = qnan<T>();
#pragma unroll
        for (int s = 0; s < C; s++) {
            const int j = q + G * s;
            if (j < N) {
#pragma unroll
                for (int m = 0; m < N; m++)
                    grp::st(CONTIG ? reinterpret_cast<V*>(Xrow) + (m * N + G * s)
                                   : reinterpret_cast<V*>(Xrow + uint64_t(uint32_t(m * N + G * s)) * seX),
                            inf ? mk<T>(nan, nan) : col[s][m]);
            }
        }
        if (q == 0) info[b] = inf;
    }
}

// k_grp_solve -- SURVEY §8(f) f1 with the lane-group mapping (c64, n = 9..16 with 4 lanes per
// system, n = 32 with 16): the factorisation of k_grp (grp_factor), then the two O(n^2) sweeps
// on the lane-distributed columns -- lane q holds y_j, then b_j / w_j, then x_j for its columns
// j = q + G*s:
//   forward  R* b = y (eq. 6; LDL R* z = y, w = D^-1 z, eq. 13): step k, the owner of column k
//            finalises b_k and broadcasts it by shuffle; each lane updates its y_j, j > k, with
//            conj(r_kj) b_k -- r_kj is row k of its own register column;
//   backward R x = b (eq. 7; LDL R x = w, eq. 14): step k (descending), each lane forms its share
//            sum_{own j > k} r_kj x_j from its register column, the G lanes combine it by
//            shuffles, and the owner of column k finalises x_k.
template <typename T, int N, int GG, bool LDL>
__global__ void __launch_bounds__(GrpShape<T, N, GG>::THREADS, GrpShape<T, N, GG>::MIN_BLOCKS)
k_grp_solve(int64_t batch, const cplx<T>* __restrict__ A, int64_t sAm, int64_t sAe,
            const cplx<T>* __restrict__ Y, int64_t sYm, int64_t sYe, cplx<T>* Xv, int64_t sXm, int64_t sXe,
            int32_t* __restrict__ info)
{
    using Sh = GrpShape<T, N, GG>;
    using V = cplx<T>;
    constexpr int G = Sh::G, C = Sh::C;
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(16) unsigned char smem_raw[];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane & (G - 1), g = lane / G;
    const int mloc = warp * Sh::MPW + g;
    int64_t b = int64_t(blockIdx.x) * Sh::MPC + mloc;
    const bool valid = b < batch;
    b = valid ? b : batch - 1;                        // the tail recomputes (never stores) the last system
    unsigned char* mbase = smem_raw + size_t(Sh::slot(mloc)) * Sh::MSTR_FULL_B;
    V* Rs = reinterpret_cast<V*>(mbase);
    T* invs = reinterpret_cast<T*>(Rs + Sh::RSZ + 2 * Sh::RB);

    V yv[C];
#pragma unroll
    for (int s = 0; s < C; s++) {
        const int j = q + G * s;
        yv[s] = (j < N) ? Y[b * sYm + int64_t(j) * sYe] : czero<T>();
    }
    V col[C][N];
    const int inf = grp_factor<T, N, GG, LDL>(col, A + b * sAm, sAe, q, Rs, invs);
    __syncwarp();

    // ---- forward: R* b = y (Cholesky b_k = y'_k / r_kk; LDL z_k = y'_k, w_k = z_k / d_k)
#pragma unroll
    for (int k = 0; k < N; k++) {
        const int qk = k % G, sk = k / G;
        const T ik = invs[k];
        V bk = yv[sk];                                   // owner's finished y'_k
        if (!LDL) bk = cscale(bk, ik);
        bk = mk<T>(__shfl_sync(FULL, bk.x, qk, G), __shfl_sync(FULL, bk.y, qk, G));
        if (q == qk) yv[sk] = LDL ? cscale(bk, ik) : bk;   // b_k (LDL: w_k)
#pragma unroll
        for (int s = 0; s < C; s++) {
            const int j = q + G * s;
            if (G * s + G - 1 > k && j > k) {            // y'_j -= conj(r_kj) b_k
                const V r = col[s][k];
                V y = yv[s];
                y.x = fmaf(-r.x, bk.x, y.x); y.x = fmaf(-r.y, bk.y, y.x);
                y.y = fmaf(-r.x, bk.y, y.y); y.y = fmaf(r.y, bk.x, y.y);
                yv[s] = y;
            }
        }
    }
    // ---- backward: R x = b (Cholesky x_k = (b_k - sum) / r_kk; LDL x_k = w_k - sum)
#pragma unroll
    for (int k = N - 1; k >= 0; k--) {
        const int qk = k % G, sk = k / G;
        V p = czero<T>();
#pragma unroll
        for (int s = 0; s < C; s++) {
            const int j = q + G * s;
            if (G * s + G - 1 > k && j > k) {            // r_kj x_j over this lane's columns
                const V r = col[s][k], x = yv[s];
                p.x = fmaf(r.x, x.x, p.x); p.x = fmaf(-r.y, x.y, p.x);
                p.y = fmaf(r.x, x.y, p.y); p.y = fmaf(r.y, x.x, p.y);
            }
        }
#pragma unroll
        for (int off = 1; off < G; off <<= 1) {
            p.x += __shfl_xor_sync(FULL, p.x, off, G);
            p.y += __shfl_xor_sync(FULL, p.y, off, G);
        }
        if (q == qk) {
            const V w = yv[sk];
            const V d = mk<T>(w.x - p.x, w.y - p.y);
            yv[sk] = LDL ? d : cscale(d, invs[k]);
        }
    }
    if (valid) {
        const T nan = qnan<T>();
#pragma unroll
        for (int s = 0; s < C; s++) {
            const int j = q + G * s;
            if (j < N) Xv[b * sXm + int64_t(j) * sXe] = inf ? mk<T>(nan, nan) : yv[s];
        }
        if (q == 0) info[b] = inf;
    }
}

}  // namespace hpdinv
