// k_lane_c64.cu -- c64 instantiations and launcher of the lane-group kernel (k_lane.cuh).
#include "dispatch.h"
#include "k_lane.cuh"

#ifndef HPDINV_G32
#define HPDINV_G32 16   // lanes per matrix for n = 25..32
#endif

namespace hpdinv {

template <bool LDL>
static int launch_lane_c64(const LaunchArgs& a) {
    using T = float;
    using fn_t = void (*)(int64_t, const cplx<T>*, int64_t, int64_t, cplx<T>*, int64_t, int64_t, int32_t*);
    fn_t fn = nullptr;
    size_t smem = 0;
    int mpc = 1;
#define HPDINV_LANE(NN, GG)                              \
    case NN:                                             \
        fn = k_lane<T, NN, GG, LDL>;                     \
        smem = LaneShape<T, NN, GG>::smem_bytes;         \
        mpc = LaneShape<T, NN, GG>::MPC;                 \
        break;
    switch (a.n) {
        HPDINV_LANE(9, 4) HPDINV_LANE(10, 4) HPDINV_LANE(11, 4) HPDINV_LANE(12, 4)
        HPDINV_LANE(13, 4) HPDINV_LANE(14, 4) HPDINV_LANE(15, 4) HPDINV_LANE(16, 4)
        HPDINV_LANE(17, 8) HPDINV_LANE(18, 8) HPDINV_LANE(19, 8) HPDINV_LANE(20, 8)
        HPDINV_LANE(21, 8) HPDINV_LANE(22, 8) HPDINV_LANE(23, 8) HPDINV_LANE(24, 8)
        HPDINV_LANE(25, HPDINV_G32) HPDINV_LANE(26, HPDINV_G32) HPDINV_LANE(27, HPDINV_G32) HPDINV_LANE(28, HPDINV_G32)
        HPDINV_LANE(29, HPDINV_G32) HPDINV_LANE(30, HPDINV_G32) HPDINV_LANE(31, HPDINV_G32) HPDINV_LANE(32, HPDINV_G32)
        default: break;
    }
#undef HPDINV_LANE
    if (!fn) return kNoKernel;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(fn), smem);
    if (e != cudaSuccess) return int(e);
    const int64_t blocks = (a.batch + mpc - 1) / mpc;
    fn<<<unsigned(blocks), 128, smem, a.stream>>>(a.batch, static_cast<const cplx<T>*>(a.A), a.sAm, a.sAe,
                                                  static_cast<cplx<T>*>(a.X), a.sXm, a.sXe, a.info);
    return int(cudaGetLastError());
}

int launch_lane_dtype0(bool ldl, const LaunchArgs& a) {
    return ldl ? launch_lane_c64<true>(a) : launch_lane_c64<false>(a);
}

}  // namespace hpdinv
