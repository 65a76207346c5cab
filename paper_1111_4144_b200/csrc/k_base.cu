// k_base.cu -- instantiations and launchers of the existing-method kernels (k_base.cuh).
#include "dispatch.h"
#include "k_base.cuh"

namespace hpdinv {

template <typename T, int METHOD>
static int launch_base_t(const LaunchArgs& a) {
    using V = cplx<T>;
    using fn_t = void (*)(int64_t, const V*, int64_t, int64_t, V*, int64_t, int64_t, int32_t*);
    fn_t fn = nullptr;
    switch (a.n) {
        case 1: fn = k_base_reg<T, 1, METHOD>; break;
        case 2: fn = k_base_reg<T, 2, METHOD>; break;
        case 3: fn = k_base_reg<T, 3, METHOD>; break;
        case 4: fn = k_base_reg<T, 4, METHOD>; break;
        case 5: fn = k_base_reg<T, 5, METHOD>; break;
        case 6: fn = k_base_reg<T, 6, METHOD>; break;
        case 7: if constexpr (sizeof(T) == 4) fn = k_base_reg<T, 7, METHOD>; break;
        case 8: if constexpr (sizeof(T) == 4) fn = k_base_reg<T, 8, METHOD>; break;
        default: break;
    }
    const V* A = static_cast<const V*>(a.A);
    V* X = static_cast<V*>(a.X);
    if (fn) {
        const int64_t blocks = (a.batch + kRegThreads - 1) / kRegThreads;
        fn<<<unsigned(blocks), kRegThreads, 0, a.stream>>>(a.batch, A, a.sAm, a.sAe, X, a.sXm, a.sXe, a.info);
        return int(cudaGetLastError());
    }
    auto gfn = k_base_gen<T, METHOD>;
    const size_t smem = base_gen_smem_bytes<T>(a.n);
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(gfn), smem);
    if (e != cudaSuccess) return int(e);
    const int64_t grid = a.batch < (int64_t(1) << 30) ? a.batch : (int64_t(1) << 30);
    gfn<<<unsigned(grid), kBaseGenThreads, smem, a.stream>>>(a.batch, a.n, A, a.sAm, a.sAe, X, a.sXm, a.sXe, a.info);
    return int(cudaGetLastError());
}

int launch_base(int method, int dtype, const LaunchArgs& a) {
    if (method == 2) return dtype == 0 ? launch_base_t<float, 2>(a) : launch_base_t<double, 2>(a);
    if (method == 3) return dtype == 0 ? launch_base_t<float, 3>(a) : launch_base_t<double, 3>(a);
    return kNoKernel;
}

const char* base_kernel_name(int method, int dtype, int n) {
    static const char* names[2][2][2] = {
        {{"k_base_reg<c64,eqsolve>", "k_base_reg<c64,trimat>"}, {"k_base_reg<c128,eqsolve>", "k_base_reg<c128,trimat>"}},
        {{"k_base_gen<c64,eqsolve>", "k_base_gen<c64,trimat>"}, {"k_base_gen<c128,eqsolve>", "k_base_gen<c128,trimat>"}},
    };
    if (method != 2 && method != 3) return nullptr;
    return names[n <= reg_max_n(dtype) ? 0 : 1][dtype][method - 2];
}

}  // namespace hpdinv
