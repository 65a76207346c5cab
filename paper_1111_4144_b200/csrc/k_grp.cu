// k_grp.cu -- instantiations and launcher of the in-place lane-group kernel (k_grp.cuh),
// selected for interleaved (SoA) inputs at n = 9..16 (complex64).
#include "dispatch.h"
#include "k_grp.cuh"

#ifndef HPDINV_G16
#define HPDINV_G16 4          // lanes per matrix at n = 16
#endif

namespace hpdinv {

template <typename T, bool LDL>
static int launch_grp_t(const LaunchArgs& a) {
    using fn_t = void (*)(int64_t, const cplx<T>*, int64_t, int64_t, cplx<T>*, int64_t, int64_t, int32_t*);
    fn_t fn = nullptr;
    size_t smem = 0;
    int mpc = 1, threads = 0;
#define HPDINV_GRP(NN, GG)                          \
    case NN:                                        \
        fn = k_grp<T, NN, GG, LDL>;                 \
        smem = GrpShape<T, NN, GG>::smem_bytes;     \
        mpc = GrpShape<T, NN, GG>::MPC;             \
        threads = GrpShape<T, NN, GG>::THREADS;     \
        break;
    if constexpr (sizeof(T) == 4) {
        switch (a.n) {
            HPDINV_GRP(9, 4) HPDINV_GRP(10, 4) HPDINV_GRP(11, 4) HPDINV_GRP(12, 4)
            HPDINV_GRP(13, 4) HPDINV_GRP(14, 4) HPDINV_GRP(15, 4) HPDINV_GRP(16, HPDINV_G16)
            HPDINV_GRP(32, 16)     // (32 lanes per matrix measured 10.3-13.1 ms at cfg5: SIMT imbalance)
            default: break;
        }
    }
#undef HPDINV_GRP
    // plane strides in bytes must fit the kernel's 32-bit address offsets (any SoA array with
    // n >= 9 that fits in device memory does)
    if (!grp_strides_ok(a.sAe, a.sXe, sizeof(cplx<T>))) fn = nullptr;
    if (!fn) return kNoKernel;
#ifndef HPDINV_GRP_NO_CONTIG
    // contiguous matrices (sAe = sXe = 1, the AoS layout of cfg5): compile-time element offsets
    if (a.n == 32 && a.sAe == 1 && a.sXe == 1) fn = k_grp<T, 32, 16, LDL, false, true>;
#endif
#ifndef HPDINV_GRP_NO_STAGE
    // staged global I/O (bulk copies of whole CTA plane segments, k_grp.cuh STG): interleaved A
    // and X with even plane strides and 16-byte aligned bases, n <= 16
    const bool stg = a.n <= 16 && a.sAm == 1 && a.sXm == 1 && a.sAe % 2 == 0 && a.sXe % 2 == 0 &&
                     (reinterpret_cast<uintptr_t>(a.A) & 15) == 0 && (reinterpret_cast<uintptr_t>(a.X) & 15) == 0;
    if (stg) {
        switch (a.n) {
#define HPDINV_GRP_STG(NN)                                   \
            case NN:                                         \
                fn = k_grp<T, NN, 4, LDL, true>;             \
                smem = GrpShape<T, NN, 4>::smem_bytes_staged; \
                break;
            HPDINV_GRP_STG(9) HPDINV_GRP_STG(10) HPDINV_GRP_STG(11) HPDINV_GRP_STG(12)
            HPDINV_GRP_STG(13) HPDINV_GRP_STG(14) HPDINV_GRP_STG(15) HPDINV_GRP_STG(16)
#undef HPDINV_GRP_STG
            default: break;
        }
    }
#endif
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(fn), smem);
    if (e != cudaSuccess) return int(e);
    const int64_t blocks = (a.batch + mpc - 1) / mpc;
    fn<<<unsigned(blocks), threads, smem, a.stream>>>(a.batch, static_cast<const cplx<T>*>(a.A), a.sAm, a.sAe,
                                                     static_cast<cplx<T>*>(a.X), a.sXm, a.sXe, a.info);
    return int(cudaGetLastError());
}

template <typename T, bool LDL>
static int launch_grp_solve_t(const SolveArgs& a) {
    using V = cplx<T>;
    using fn_t = void (*)(int64_t, const V*, int64_t, int64_t, const V*, int64_t, int64_t, V*, int64_t, int64_t, int32_t*);
    fn_t fn = nullptr;
    size_t smem = 0;
    int mpc = 1, threads = 0;
#define HPDINV_GRPS(NN, GG)                         \
    case NN:                                        \
        fn = k_grp_solve<T, NN, GG, LDL>;           \
        smem = GrpShape<T, NN, GG>::smem_bytes_full; \
        mpc = GrpShape<T, NN, GG>::MPC;             \
        threads = GrpShape<T, NN, GG>::THREADS;     \
        break;
    if constexpr (sizeof(T) == 4) {
        switch (a.n) {
            HPDINV_GRPS(9, 4) HPDINV_GRPS(10, 4) HPDINV_GRPS(11, 4) HPDINV_GRPS(12, 4)
            HPDINV_GRPS(13, 4) HPDINV_GRPS(14, 4) HPDINV_GRPS(15, 4) HPDINV_GRPS(16, 4)
            HPDINV_GRPS(32, 16)
            default: break;
        }
    }
#undef HPDINV_GRPS
    if (!grp_strides_ok(a.sAe, 0, sizeof(V))) fn = nullptr;
    if (!fn) return kNoKernel;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(fn), smem);
    if (e != cudaSuccess) return int(e);
    const int64_t blocks = (a.batch + mpc - 1) / mpc;
    fn<<<unsigned(blocks), threads, smem, a.stream>>>(a.batch, static_cast<const V*>(a.A), a.sAm, a.sAe,
                                                     static_cast<const V*>(a.Y), a.sYm, a.sYe,
                                                     static_cast<V*>(a.X), a.sXm, a.sXe, a.info);
    return int(cudaGetLastError());
}

bool grp_solve_accepts(int dtype, int n, int64_t sAe) {
    return dtype == 0 && ((n >= 9 && n <= 16) || n == 32) && grp_strides_ok(sAe, 0, 8);
}

int launch_grp_solve(int dtype, bool ldl, const SolveArgs& a) {
    if (dtype != 0) return kNoKernel;
    return ldl ? launch_grp_solve_t<float, true>(a) : launch_grp_solve_t<float, false>(a);
}

int launch_grp(int dtype, bool ldl, const LaunchArgs& a) {
    if (dtype == 0) return ldl ? launch_grp_t<float, true>(a) : launch_grp_t<float, false>(a);
    return kNoKernel;
}

}  // namespace hpdinv
