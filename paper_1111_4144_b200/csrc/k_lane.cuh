// k_lane.cuh -- G lanes per matrix ("lane group"), 32/G matrices per warp, for mid-size n
// (c64 9..24, c128 7..16).  The n columns of a matrix are dealt cyclically to the G lanes:
// lane q of a group owns columns j = q + G*s, s = 0..C-1, so every lane of the group has
// nearly the same number of active columns at every step of the triangular recursions.
//
//   S1  each lane loads the upper part of its columns (a_lj, l <= j) into registers;
//   S2  right-looking Cholesky (eqs. 3-4) / LDL (eqs. 10-11): at step i the owner of column
//       i forms the pivot, broadcasts 1/r_ii (1/d_i) by shuffle, every lane scales its
//       entries of row i of R and writes them to a per-matrix row store in shared memory,
//       then updates its columns a'_lj -= conj(r_il) r_ij (LDL: conj(r_il) d_i r_ij, which
//       is conj(r_il) times the unscaled a'_ij) reading row i back by broadcast;
//   S3  S = diag(1/r_kk) (eq. 24) / S~ = diag(1/d_k) (eq. 29): the broadcast reciprocals;
//   S4  rows k = n-1..0 of X (eqs. 22-24, App. A.1 order): lane j accumulates
//       sum_{m>k} r_km x~_mj over its FULL register column of the trailing block, the new
//       row is gathered into the owner of column k through a shared row buffer (it becomes
//       that column's lower part, x_mk = conj(x_km)), and x_kk is formed real from a
//       G-lane shuffle reduction of Re(r_km conj(x_km));
//   S5  every lane stores its columns; the lower half is the bitwise conjugate (mirror).
#pragma once
#include "cplx.cuh"

namespace hpdinv {

template <typename T, int N, int G>
struct LaneShape {
    static constexpr int C = (N + G - 1) / G;     // columns per lane
    static constexpr int MPW = 32 / G;             // matrices per warp
    static constexpr int WARPS = 4;
    static constexpr int MPC = MPW * WARPS;        // matrices per CTA
    static constexpr int P = sizeof(T) == 4 ? 2 : 1;   // complex elements per 16-byte access
    __host__ __device__ static constexpr int rlen(int i) { return ((N - i) + P - 1) / P * P; }
    __host__ __device__ static constexpr int roff(int i) { int o = 0; for (int k = 0; k < i; k++) o += rlen(k); return o; }
    static constexpr int RSZ = roff(N);
    static constexpr int ESZ = int(sizeof(cplx<T>));
    // per-matrix stride (elements): R rows + a row buffer, padded so that the stride in bytes
    // is 16 mod 128: the MPW groups of a warp then read distinct 16-byte bank quads.
    static constexpr int raw_bytes = (RSZ + N + G) * ESZ;   // row buffer has G spare slots
    static constexpr int MSTR = (((raw_bytes + 127) / 128) * 128 + 16) / ESZ;
    static constexpr size_t smem_bytes = size_t(MPC) * MSTR * ESZ;
};

// Fetch complex element `o` (0-based offset inside a 16-byte-aligned row) as part of the
// 16-byte vector that holds it; for fp32 the pair (o & ~1, o | 1) comes in one LDS.128.
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

template <typename T, int N, int G, bool LDL>
__global__ void __launch_bounds__(128)
k_lane(int64_t batch, const cplx<T>* __restrict__ A, int64_t sAm, int64_t sAe,
       cplx<T>* X, int64_t sXm, int64_t sXe, int32_t* __restrict__ info)
{
    using S = LaneShape<T, N, G>;
    constexpr int C = S::C, P = S::P;
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(16) unsigned char smem_raw[];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane & (G - 1), g = lane / G;
    const int mloc = warp * S::MPW + g;
    const int64_t b = int64_t(blockIdx.x) * S::MPC + mloc;
    const bool valid = b < batch;
    cplx<T>* Rs = reinterpret_cast<cplx<T>*>(smem_raw) + size_t(mloc) * S::MSTR;   // R rows
    cplx<T>* rowbuf = Rs + S::RSZ;                                                     // X row k

    // ---------------------------------------------------------------- S1: load columns
    cplx<T> a[C][N];
    {
        const cplx<T>* Ab = A + (valid ? b : 0) * sAm;
#pragma unroll
        for (int s = 0; s < C; s++) {
            const int j = q + G * s;
#pragma unroll
            for (int l = 0; l < N; l++) {
                if (l <= G * s + G - 1) {                 // static: some lane may need it
                    if (valid && l <= j && j < N) {
                        cplx<T> v = __ldg(Ab + int64_t(l * N + j) * sAe);
                        if (l == j) v.y = T(0);
                        a[s][l] = v;
                    } else {
                        a[s][l] = czero<T>();
                    }
                }
            }
        }
    }

    // -------------------------------------------------------- S2: right-looking factorisation
    T inv[N];
    int inf = 0;
#pragma unroll
    for (int i = 0; i < N; i++) {
        const int qi = i % G, si = i / G;
        // only the owner lane's value is meaningful; the others feed 1.0 so that no lane takes
        // the (called) slow path of the IEEE sqrt / reciprocal on a garbage operand
        const T t = (q == qi) ? a[si][i].x : T(1);
        T iv;
        if (LDL) iv = rcp_rn(t);
        else iv = rcp_rn(sqrt_rn(t));
        int bad = !(t > T(0));
        iv = __shfl_sync(FULL, iv, qi, G);
        bad = __shfl_sync(FULL, bad, qi, G);
        if (bad && inf == 0) inf = i + 1;
        inv[i] = iv;
        // Branch-free SIMT: every statically possible (slot, row) update is executed by all
        // lanes; for a lane whose column j is not active the update lands on storage that is
        // dead for that column (strict lower part of A, rows <= j of a finished pivot), so only
        // the shared-memory stores need a predicate.
        cplx<T> u[C];
        cplx<T>* Ri = Rs + S::roff(i);
#pragma unroll
        for (int s = 0; s < C; s++) {
            const int j = q + G * s;
            if (G * s + G - 1 > i) {
                u[s] = a[s][i];
                const cplx<T> r = cscale(u[s], iv);
                a[s][i] = r;
                if (j > i) Ri[j - i] = r;
            }
        }
        __syncwarp();
#pragma unroll
        for (int o = 0; o < N; o += P) {
            if (o >= N - i) continue;
            cplx<T> e[2];
            lds_pair<T>(Ri, o, e[0], e[1]);
#pragma unroll
            for (int h = 0; h < P; h++) {
                const int l = i + o + h;
                if (l > i && l < N) {
#pragma unroll
                    for (int s = 0; s < C; s++) {
                        if (G * s + G - 1 >= l) cfms_conj(a[s][l], e[h], LDL ? u[s] : a[s][i]);
                    }
                }
            }
        }
    }

    // ------------------------------------------------ S3/S4: proposed inversion, rows k = n..1
    cplx<T> x[C][N];
#pragma unroll
    for (int s = 0; s < C; s++)
#pragma unroll
        for (int m = 0; m < N; m++) x[s][m] = czero<T>();
#pragma unroll
    for (int k = N - 1; k >= 0; k--) {
        const int qk = k % G, sk = k / G;
        const cplx<T>* Rk = Rs + S::roff(k);
        cplx<T> acc[C], rkj[C];
#pragma unroll
        for (int s = 0; s < C; s++) { acc[s] = czero<T>(); rkj[s] = czero<T>(); }
#pragma unroll
        for (int o = 0; o < N; o += P) {
            if (o >= N - k) continue;
            cplx<T> e[2];
            lds_pair<T>(Rk, o, e[0], e[1]);
#pragma unroll
            for (int h = 0; h < P; h++) {
                const int l = k + o + h;
                if (l > k && l < N) {
#pragma unroll
                    for (int s = 0; s < C; s++) {
                        if (G * s + G - 1 > k) {
                            cfma(acc[s], e[h], x[s][l]);
                            if (l >= G * s && l <= G * s + G - 1) {
                                const bool hit = (q + G * s) == l;
                                rkj[s].x = hit ? e[h].x : rkj[s].x;
                                rkj[s].y = hit ? e[h].y : rkj[s].y;
                            }
                        }
                    }
                }
            }
        }
        T p = T(0);
#pragma unroll
        for (int s = 0; s < C; s++) {
            const int j = q + G * s;
            if (G * s + G - 1 > k) {
                // for j <= k the value is dead: x[s][k] of such a column is rewritten by the
                // gather (j < k) or by the diagonal (j == k) before it is read
                const cplx<T> xv = LDL ? mk<T>(-acc[s].x, -acc[s].y) : cscale(acc[s], -inv[k]);
                x[s][k] = xv;
                rowbuf[j] = xv;
                p = re_dot_conj(p, rkj[s], xv);         // rkj[s] == 0 unless j > k
            }
        }
#pragma unroll
        for (int off = 1; off < G; off <<= 1) p += __shfl_xor_sync(FULL, p, off, G);
        __syncwarp();
        const bool own = (q == qk);                     // this lane owns column k
#pragma unroll
        for (int o = 0; o < N; o += P) {
            if (o + P - 1 <= k) continue;
            cplx<T> e[2];
            lds_pair<T>(rowbuf, o, e[0], e[1]);          // aligned pair holding element o
#pragma unroll
            for (int h = 0; h < P; h++) {
                const int m = o + h;
                if (m > k && m < N) {
                    x[sk][m].x = own ? e[h].x : x[sk][m].x;
                    x[sk][m].y = own ? -e[h].y : x[sk][m].y;
                }
            }
        }
        const T ik = inv[k];
        const T xkk = LDL ? ik - p : ik * (ik - p);
        x[sk][k].x = own ? xkk : x[sk][k].x;
        x[sk][k].y = own ? T(0) : x[sk][k].y;
        __syncwarp();
    }

    // ------------------------------------------------------------------ S5: mirror + store
    if (valid) {
        cplx<T>* Xb = X + b * sXm;
        const T nan = qnan<T>();
#pragma unroll
        for (int s = 0; s < C; s++) {
            const int j = q + G * s;
            if (j < N) {
#pragma unroll
                for (int m = 0; m < N; m++) {
                    cplx<T> v = x[s][m];
                    if (inf) v = mk<T>(nan, nan);
                    Xb[int64_t(m * N + j) * sXe] = v;
                }
            }
        }
        if (q == 0) info[b] = inf;
    }
}

}  // namespace hpdinv
