// k_generic.cu -- instantiations and launcher of the one-matrix-per-CTA shared-memory kernel.
#include "dispatch.h"
#include "k_generic.cuh"

namespace hpdinv {

template <typename T, bool LDL>
static int launch_generic_t(const LaunchArgs& a) {
    const size_t smem = generic_smem_bytes<T>(a.n);
    auto fn = k_generic<T, LDL>;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(fn), smem);
    if (e != cudaSuccess) return int(e);
    const int64_t blocks = a.batch < (int64_t(1) << 30) ? a.batch : (int64_t(1) << 30);
    fn<<<unsigned(blocks), kGenericThreads, smem, a.stream>>>(a.batch, a.n, static_cast<const cplx<T>*>(a.A), a.sAm,
                                                            a.sAe, static_cast<cplx<T>*>(a.X), a.sXm, a.sXe, a.info);
    return int(cudaGetLastError());
}

int launch_generic(int dtype, bool ldl, const LaunchArgs& a) {
    if (dtype == 0) return ldl ? launch_generic_t<float, true>(a) : launch_generic_t<float, false>(a);
    return ldl ? launch_generic_t<double, true>(a) : launch_generic_t<double, false>(a);
}

}  // namespace hpdinv
