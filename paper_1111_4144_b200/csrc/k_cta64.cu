// k_cta64.cu -- instantiations and launcher of the n = 64 one-matrix-per-CTA kernel.
#include "dispatch.h"
#include "k_cta64.cuh"

namespace hpdinv {

template <typename T, bool LDL>
static int launch_cta64_t(const LaunchArgs& a) {
    if (a.n != 64) return kNoKernel;
    auto fn = k_cta64<T, LDL>;
    const size_t smem = Cta64Shape<T>::smem_bytes;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(fn), smem);
    if (e != cudaSuccess) return int(e);
    const int64_t blocks = a.batch < (int64_t(1) << 30) ? a.batch : (int64_t(1) << 30);
    fn<<<unsigned(blocks), kCta64Threads, smem, a.stream>>>(a.batch, static_cast<const cplx<T>*>(a.A), a.sAm, a.sAe,
                                                           static_cast<cplx<T>*>(a.X), a.sXm, a.sXe, a.info);
    return int(cudaGetLastError());
}

int launch_cta(int dtype, bool ldl, const LaunchArgs& a) {
    if (dtype == 0) return ldl ? launch_cta64_t<float, true>(a) : launch_cta64_t<float, false>(a);
    return ldl ? launch_cta64_t<double, true>(a) : launch_cta64_t<double, false>(a);
}

}  // namespace hpdinv
