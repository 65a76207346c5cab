// k_reg.cu -- instantiations and launcher of the one-matrix-per-thread kernel (k_reg.cuh).
#include "dispatch.h"
#include "k_reg.cuh"

namespace hpdinv {

template <typename T, bool LDL>
static int launch_reg_t(const LaunchArgs& a) {
    using fn_t = void (*)(int64_t, const cplx<T>*, int64_t, int64_t, cplx<T>*, int64_t, int64_t, int32_t*);
    fn_t fn = nullptr;
    switch (a.n) {
        case 1: fn = k_reg<T, 1, LDL>; break;
        case 2: fn = k_reg<T, 2, LDL>; break;
        case 3: fn = k_reg<T, 3, LDL>; break;
        case 4: fn = k_reg<T, 4, LDL>; break;
        case 5: fn = k_reg<T, 5, LDL>; break;
        case 6: fn = k_reg<T, 6, LDL>; break;
        case 7: if constexpr (sizeof(T) == 4) fn = k_reg<T, 7, LDL>; break;
        case 8: if constexpr (sizeof(T) == 4) fn = k_reg<T, 8, LDL>; break;
        default: break;
    }
    if (!fn) return kNoKernel;
    const int64_t blocks = (a.batch + kRegThreads - 1) / kRegThreads;
    fn<<<unsigned(blocks), kRegThreads, 0, a.stream>>>(a.batch, static_cast<const cplx<T>*>(a.A), a.sAm, a.sAe,
                                                      static_cast<cplx<T>*>(a.X), a.sXm, a.sXe, a.info);
    return int(cudaGetLastError());
}

int launch_reg(int dtype, bool ldl, const LaunchArgs& a) {
    if (dtype == 0) return ldl ? launch_reg_t<float, true>(a) : launch_reg_t<float, false>(a);
    return ldl ? launch_reg_t<double, true>(a) : launch_reg_t<double, false>(a);
}

}  // namespace hpdinv
