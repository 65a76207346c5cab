// k_nh.cu -- instantiations and launchers of the non-Hermitian inversion kernels (k_nh.cuh).
#include "dispatch.h"
#include "k_nh.cuh"

namespace hpdinv {

template <typename T>
static int launch_nh_t(const LaunchArgs& a) {
    using V = cplx<T>;
    using fn_t = void (*)(int64_t, const V*, int64_t, int64_t, V*, int64_t, int64_t, int32_t*);
    fn_t fn = nullptr;
    switch (a.n) {
        case 1: fn = k_nh_reg<T, 1>; break;
        case 2: fn = k_nh_reg<T, 2>; break;
        case 3: fn = k_nh_reg<T, 3>; break;
        case 4: fn = k_nh_reg<T, 4>; break;
        case 5: fn = k_nh_reg<T, 5>; break;
        case 6: fn = k_nh_reg<T, 6>; break;
        case 7: if constexpr (sizeof(T) == 4) fn = k_nh_reg<T, 7>; break;
        case 8: if constexpr (sizeof(T) == 4) fn = k_nh_reg<T, 8>; break;
        default: break;
    }
    const V* D = static_cast<const V*>(a.A);
    V* Y = static_cast<V*>(a.X);
    if (fn) {
        const size_t smem = size_t(a.n) * a.n * sizeof(V) * kRegThreads;   // D, one column per thread
        cudaError_t e = ensure_smem(reinterpret_cast<const void*>(fn), smem);
        if (e != cudaSuccess) return int(e);
        const int64_t blocks = (a.batch + kRegThreads - 1) / kRegThreads;
        fn<<<unsigned(blocks), kRegThreads, smem, a.stream>>>(a.batch, D, a.sAm, a.sAe, Y, a.sXm, a.sXe, a.info);
        return int(cudaGetLastError());
    }
    auto gfn = k_nh_gen<T>;
    const size_t smem = nh_gen_smem_bytes<T>(a.n);
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(gfn), smem);
    if (e != cudaSuccess) return int(e);
    const int64_t grid = a.batch < (int64_t(1) << 30) ? a.batch : (int64_t(1) << 30);
    gfn<<<unsigned(grid), kNhGenThreads, smem, a.stream>>>(a.batch, a.n, D, a.sAm, a.sAe, Y, a.sXm, a.sXe, a.info);
    return int(cudaGetLastError());
}

int launch_nh(int dtype, const LaunchArgs& a) {
    return dtype == 0 ? launch_nh_t<float>(a) : launch_nh_t<double>(a);
}

const char* nh_kernel_name(int dtype, int n) {
    static const char* names[2][2] = {{"k_nh_reg<c64>", "k_nh_reg<c128>"}, {"k_nh_gen<c64>", "k_nh_gen<c128>"}};
    return names[n <= reg_max_n(dtype) ? 0 : 1][dtype];
}

}  // namespace hpdinv
