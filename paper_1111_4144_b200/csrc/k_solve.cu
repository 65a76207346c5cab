// k_solve.cu -- instantiations and launchers of the batched linear-solve kernels (k_solve.cuh).
#include "dispatch.h"
#include "k_solve.cuh"

namespace hpdinv {

template <typename T, bool LDL>
static int launch_solve_t(const SolveArgs& a) {
    using V = cplx<T>;
    using fn_t = void (*)(int64_t, const V*, int64_t, int64_t, const V*, int64_t, int64_t, V*, int64_t, int64_t, int32_t*);
    fn_t fn = nullptr;
    switch (a.n) {
        case 1: fn = k_solve_reg<T, 1, LDL>; break;
        case 2: fn = k_solve_reg<T, 2, LDL>; break;
        case 3: fn = k_solve_reg<T, 3, LDL>; break;
        case 4: fn = k_solve_reg<T, 4, LDL>; break;
        case 5: fn = k_solve_reg<T, 5, LDL>; break;
        case 6: fn = k_solve_reg<T, 6, LDL>; break;
        case 7: if constexpr (sizeof(T) == 4) fn = k_solve_reg<T, 7, LDL>; break;
        case 8: if constexpr (sizeof(T) == 4) fn = k_solve_reg<T, 8, LDL>; break;
        default: break;
    }
    const V* A = static_cast<const V*>(a.A);
    const V* Y = static_cast<const V*>(a.Y);
    V* X = static_cast<V*>(a.X);
    if (fn) {
        const int64_t blocks = (a.batch + kSolveThreads - 1) / kSolveThreads;
        fn<<<unsigned(blocks), kSolveThreads, 0, a.stream>>>(a.batch, A, a.sAm, a.sAe, Y, a.sYm, a.sYe,
                                                            X, a.sXm, a.sXe, a.info);
        return int(cudaGetLastError());
    }
    // c64 n = 9..16 and 32: the lane-group solve (k_grp_solve); otherwise the CTA fallback
    if (sizeof(T) == 4) {
        const int rc = launch_grp_solve(0, LDL, a);
        if (rc != kNoKernel) return rc;
    }
    auto gfn = k_solve_gen<T, LDL>;
    const size_t smem = solve_gen_smem_bytes<T>(a.n);
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(gfn), smem);
    if (e != cudaSuccess) return int(e);
    const int64_t grid = a.batch < (int64_t(1) << 30) ? a.batch : (int64_t(1) << 30);   // grid-stride
    gfn<<<unsigned(grid), kSolveGenThreads, smem, a.stream>>>(a.batch, a.n, A, a.sAm, a.sAe, Y, a.sYm, a.sYe,
                                                             X, a.sXm, a.sXe, a.info);
    return int(cudaGetLastError());
}

int launch_solve(int dtype, bool ldl, const SolveArgs& a) {
    if (dtype == 0) return ldl ? launch_solve_t<float, true>(a) : launch_solve_t<float, false>(a);
    return ldl ? launch_solve_t<double, true>(a) : launch_solve_t<double, false>(a);
}

const char* solve_kernel_name(int dtype, bool ldl, int n) {
    static const char* names[2][2][2] = {
        {{"k_solve_reg<c64,chol>", "k_solve_reg<c64,ldl>"}, {"k_solve_reg<c128,chol>", "k_solve_reg<c128,ldl>"}},
        {{"k_solve_gen<c64,chol>", "k_solve_gen<c64,ldl>"}, {"k_solve_gen<c128,chol>", "k_solve_gen<c128,ldl>"}},
    };
    const bool reg = n <= reg_max_n(dtype);
    if (!reg && dtype == 0 && ((n >= 9 && n <= 16) || n == 32))
        return ldl ? "k_grp_solve<c64,ldl>" : "k_grp_solve<c64,chol>";
    return names[reg ? 0 : 1][dtype][ldl ? 1 : 0];
}

}  // namespace hpdinv
