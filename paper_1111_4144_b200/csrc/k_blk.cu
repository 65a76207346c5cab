// k_blk.cu -- instantiations and launcher of the blocked one-matrix-per-CTA kernel (k_blk.cuh):
// n = 32 (one warp per matrix) and n = 64 (four warps per matrix), both dtypes, both methods.
#include "dispatch.h"
#include "k_blk.cuh"

namespace hpdinv {

template <typename T, int N, int NB, bool LDL, int NT, int RT>
static int launch_blk_t(const LaunchArgs& a) {
    using Sh = BlkShape<T, N, NB, NT, RT>;
    auto fn = k_blk<T, N, NB, LDL, NT, RT>;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(fn), Sh::smem_bytes);
    if (e != cudaSuccess) return int(e);
    const int64_t lim = int64_t(1) << 31;
    for (int64_t b0 = 0; b0 < a.batch; b0 += lim - 1) {       // grid.x limit
        const int64_t nb = (a.batch - b0) < (lim - 1) ? (a.batch - b0) : (lim - 1);
        const cplx<T>* A = static_cast<const cplx<T>*>(a.A) + b0 * a.sAm;
        cplx<T>* X = static_cast<cplx<T>*>(a.X) + b0 * a.sXm;
        fn<<<unsigned(nb), NT, Sh::smem_bytes, a.stream>>>(nb, A, a.sAm, a.sAe, X, a.sXm, a.sXe, a.info + b0);
        if ((e = cudaGetLastError()) != cudaSuccess) return int(e);
    }
    return 0;
}

#ifndef HPDINV_BLK_NB32
#define HPDINV_BLK_NB32 8      // panel height at n = 32
#endif
#ifndef HPDINV_BLK_NB64
#define HPDINV_BLK_NB64 8      // panel height at n = 64
#endif
#ifndef HPDINV_BLK_NT64
#define HPDINV_BLK_NT64 128    // threads per matrix at n = 64
#endif

template <bool LDL>
static int launch_blk_m(int dtype, const LaunchArgs& a) {
    if (dtype == 0) {
        if (a.n == 32) return launch_blk_t<float, 32, HPDINV_BLK_NB32, LDL, 32, 2>(a);
        if (a.n == 64) return launch_blk_t<float, 64, HPDINV_BLK_NB64, LDL, HPDINV_BLK_NT64, 2>(a);
    } else {
        if (a.n == 32) return launch_blk_t<double, 32, HPDINV_BLK_NB32, LDL, 32, 2>(a);
        if (a.n == 64) return launch_blk_t<double, 64, HPDINV_BLK_NB64, LDL, HPDINV_BLK_NT64, 2>(a);
    }
    return kNoKernel;
}

int launch_blk(int dtype, bool ldl, const LaunchArgs& a) {
    return ldl ? launch_blk_m<true>(dtype, a) : launch_blk_m<false>(dtype, a);
}

}  // namespace hpdinv
