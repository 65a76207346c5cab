// dispatch.h -- internal (not part of the C ABI): per-family launchers, one translation unit
// per kernel family so the sm_100a instantiations compile in parallel.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace hpdinv {

struct LaunchArgs {
    int64_t batch;
    int n;
    const void* A;
    int64_t sAm, sAe;
    void* X;
    int64_t sXm, sXe;
    int32_t* info;
    cudaStream_t stream;
};

// Batched solve A_b x_b = y_b: vectors at base[b*s?m + i*s?e].
struct SolveArgs {
    int64_t batch;
    int n;
    const void* A;
    int64_t sAm, sAe;
    const void* Y;
    int64_t sYm, sYe;
    void* X;
    int64_t sXm, sXe;
    int32_t* info;
    cudaStream_t stream;
};

constexpr int kNoKernel = -1000;   // launcher has no instantiation for this n

// Each returns 0 / cudaError_t of the launch, or kNoKernel.
int launch_reg(int dtype, bool ldl, const LaunchArgs& a);       // k_reg.cu
int launch_lane(int dtype, bool ldl, const LaunchArgs& a);      // k_lane_c64.cu / k_lane_c128.cu
int launch_generic(int dtype, bool ldl, const LaunchArgs& a);   // k_generic.cu
int launch_grp(int dtype, bool ldl, const LaunchArgs& a);       // k_grp.cu (interleaved, c64 9..16)
int launch_blk(int dtype, bool ldl, const LaunchArgs& a);       // k_blk.cu (n = 32, 64)
int launch_dmma(const LaunchArgs& a);                            // k_dmma.cu (c128, n = 64, Cholesky, AoS A)
bool dmma_accepts(int dtype, bool ldl, int n, int64_t sAm, int64_t sAe);
int launch_solve(int dtype, bool ldl, const SolveArgs& a);      // k_solve.cu (any n <= 64)
int launch_grp_solve(int dtype, bool ldl, const SolveArgs& a);  // k_grp.cu (c64 n = 9..16, 32)
bool grp_solve_accepts(int dtype, int n, int64_t sAe);
const char* solve_kernel_name(int dtype, bool ldl, int n);
int launch_base(int method, int dtype, const LaunchArgs& a);    // k_base.cu (methods 2, 3)
const char* base_kernel_name(int method, int dtype, int n);
int launch_nh(int dtype, const LaunchArgs& a);                  // k_nh.cu (non-Hermitian, f2)
const char* nh_kernel_name(int dtype, int n);

// Largest n of each family per dtype (0 = c64, 1 = c128).
constexpr int reg_max_n(int dtype) { return dtype == 0 ? 8 : 6; }
constexpr int lane_max_n(int dtype) { return dtype == 0 ? 32 : 16; }
constexpr int grp_max_n(int dtype) { return dtype == 0 ? 16 : 0; }

// k_grp addresses element planes with 32-bit byte offsets: it takes SoA plane strides below 4 GiB
// (the launcher declines otherwise and the dispatcher falls back to k_lane)
constexpr bool grp_strides_ok(int64_t sAe, int64_t sXe, size_t elem) {
    return uint64_t(sAe) * elem < (uint64_t(1) << 32) && uint64_t(sXe) * elem < (uint64_t(1) << 32);
}

// Raise the dynamic shared-memory limit of `fn` on the current device once (thread-safe).
cudaError_t ensure_smem(const void* fn, size_t bytes);

}  // namespace hpdinv
