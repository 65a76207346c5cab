// k_dmma.cu -- launcher of the FP64-tensor-core kernel (k_dmma.cuh): complex128, n = 64,
// Cholesky, contiguous (AoS) A.  Builds the TMA tensor map of A per call (the driver's
// cuTensorMapEncodeTiled, reached through cudaGetDriverEntryPoint so the library needs no
// -lcuda).  Declines (kNoKernel -> the dispatcher falls back to k_blk) for any other shape.
#include <mutex>

#include <cuda.h>

#include "dispatch.h"
#include "k_dmma.cuh"

namespace hpdinv {

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}
}  // namespace

bool dmma_accepts(int dtype, bool ldl, int n, int64_t sAm, int64_t sAe) {
    return dtype == 1 && !ldl && n == dm::N && sAe == 1 && sAm >= int64_t(dm::N) * dm::N;
}

int launch_dmma(const LaunchArgs& a) {
    if (a.n != dm::N || a.sAe != 1) return kNoKernel;
    EncodeTiledFn enc = encode_fn();
    if (!enc) return kNoKernel;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k_dmma), dm::SMEM);
    if (e != cudaSuccess) return int(e);
    const int64_t lim = (int64_t(1) << 31) - 1;                 // grid.x and the map's z extent
    for (int64_t b0 = 0; b0 < a.batch; b0 += lim) {
        const int64_t nb = (a.batch - b0) < lim ? (a.batch - b0) : lim;
        const double2* A = static_cast<const double2*>(a.A) + b0 * a.sAm;
        double2* X = static_cast<double2*>(a.X) + b0 * a.sXm;
        CUtensorMap tm;
        const cuuint64_t dims[3] = {cuuint64_t(2 * dm::N), cuuint64_t(dm::N), cuuint64_t(nb)};
        const cuuint64_t strides[2] = {cuuint64_t(dm::N) * 16, cuuint64_t(a.sAm) * 16};   // bytes
        const cuuint32_t box[3] = {16, 8, 1};                                              // one 8x8 tile
        const cuuint32_t estr[3] = {1, 1, 1};
        const CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(A), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return b0 == 0 ? kNoKernel : int(cudaErrorInvalidValue);
        // X by TMA bulk stores when it is contiguous row-major per matrix (else per-lane stores)
        CUtensorMap tmx;
        int xtma = 0;
        if (a.sXe == 1 && (reinterpret_cast<uintptr_t>(X) & 15) == 0) {
            const cuuint64_t xstr[2] = {cuuint64_t(dm::N) * 16, cuuint64_t(a.sXm) * 16};
            xtma = enc(&tmx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, X, dims, xstr, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
        if (!xtma) tmx = tm;
        // persistent: one CTA of WPB warps per SM (WPB matrices in flight per SM)
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t need = (nb + dm::WPB - 1) / dm::WPB;
        const unsigned grid = unsigned(need < sms ? need : sms);
        k_dmma<<<grid, dm::NT, dm::SMEM, a.stream>>>(tm, tmx, xtma, nb, X, a.sXm, a.sXe, a.info + b0);
        if ((e = cudaGetLastError()) != cudaSuccess) return int(e);
    }
    return 0;
}

}  // namespace hpdinv
