// api.cu -- the C ABI of include/hpdinv.h: argument validation, layout classification and
// kernel-family selection per (method, dtype, n).  Host code only; the kernel families live
// in their own translation units (k_reg.cu, k_lane_c64.cu, k_lane_c128.cu, k_generic.cu).
#include <cstdlib>
#include <mutex>
#include <map>
#include <utility>

#include "../../include/hpdinv.h"
#include "dispatch.h"

namespace hpdinv {

int launch_lane_dtype0(bool ldl, const LaunchArgs& a);
int launch_lane_dtype1(bool ldl, const LaunchArgs& a);

int launch_lane(int dtype, bool ldl, const LaunchArgs& a) {
    return dtype == 0 ? launch_lane_dtype0(ldl, a) : launch_lane_dtype1(ldl, a);
}

cudaError_t ensure_smem(const void* fn, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;   // (kernel, device) -> bytes set
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    auto it = done.find({fn, dev});
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    if (e != cudaSuccess) return e;
    // tuning experiment: HPDINV_SMEM_CARVEOUT=<percent> sets the preferred shared-memory
    // carveout of the large-smem kernels (unset: the driver's choice)
    if (const char* cv = getenv("HPDINV_SMEM_CARVEOUT")) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
        if (e != cudaSuccess) return e;
    }
    done[{fn, dev}] = bytes;
    return e;
}

}  // namespace hpdinv

using namespace hpdinv;

namespace {

enum LayoutClass { kInvalid = -1, kSoA = 0, kAoS = 1 };

LayoutClass classify(int64_t batch, int n, int64_t sm, int64_t se) {
    if (sm < 1 || se < 1) return kInvalid;
    if (n == 1) return sm == 1 ? kSoA : kAoS;
    if (sm == 1 && se >= batch) return kSoA;
    if (se == 1 && sm >= int64_t(n) * n) return kAoS;
    return kInvalid;
}

enum Family { kReg, kLane, kGeneric, kGrp, kBlk };

// interleaved A and X at n = 9..16 (c64): in-place lane groups (k_grp); otherwise the general
// lane-group kernel (k_lane)
Family family(int dtype, int n, bool soa) {
    if (n <= reg_max_n(dtype)) return kReg;
    if (soa && dtype == 0 && n <= grp_max_n(dtype)) return kGrp;
    if (dtype == 0 && n == 32) return kGrp;            // 16 lanes per matrix, either layout
    if (n == 32 || n == 64) return kBlk;
    if (n <= lane_max_n(dtype)) return kLane;
    return kGeneric;
}

const char* family_name(Family f, int dtype, bool ldl) {
    static const char* names[5][2][2] = {
        {{"k_reg<c64,chol>", "k_reg<c64,ldl>"}, {"k_reg<c128,chol>", "k_reg<c128,ldl>"}},
        {{"k_lane<c64,chol>", "k_lane<c64,ldl>"}, {"k_lane<c128,chol>", "k_lane<c128,ldl>"}},
        {{"k_generic<c64,chol>", "k_generic<c64,ldl>"}, {"k_generic<c128,chol>", "k_generic<c128,ldl>"}},
        {{"k_grp<c64,chol>", "k_grp<c64,ldl>"}, {"k_grp<c128,chol>", "k_grp<c128,ldl>"}},
        {{"k_blk<c64,chol>", "k_blk<c64,ldl>"}, {"k_blk<c128,chol>", "k_blk<c128,ldl>"}},
    };
    return names[f][dtype][ldl ? 1 : 0];
}

int validate(const LaunchArgs& c, size_t elem_bytes) {
    if (c.batch < 0) return -1;
    if (c.n < 1 || c.n > HPDINV_MAX_N) return -2;
    if (c.batch == 0) return 0;
    if (!c.A) return -3;
    if (classify(c.batch, c.n, c.sAm, c.sAe) == kInvalid) return -4;
    if (!c.X) return -6;
    if (classify(c.batch, c.n, c.sXm, c.sXe) == kInvalid) return -7;
    if (!c.info) return -9;
    if (reinterpret_cast<uintptr_t>(c.A) % elem_bytes) return -3;
    if (reinterpret_cast<uintptr_t>(c.X) % elem_bytes) return -6;
    if (reinterpret_cast<uintptr_t>(c.info) % 4) return -9;
    return 1;
}

int run(int dtype, bool ldl, const LaunchArgs& c) {
    const int v = validate(c, dtype == 0 ? 8 : 16);
    if (v <= 0) return v;
    int rc = kNoKernel;
    const bool soa = classify(c.batch, c.n, c.sAm, c.sAe) == kSoA && classify(c.batch, c.n, c.sXm, c.sXe) == kSoA;
    // complex128 n = 64 Cholesky with a contiguous A: the FP64 tensor-core kernel (k_dmma)
    if (dmma_accepts(dtype, ldl, c.n, c.sAm, c.sAe)) {
        rc = launch_dmma(c);
        if (rc != kNoKernel) return rc;
    }
    switch (family(dtype, c.n, soa)) {
        case kReg: rc = launch_reg(dtype, ldl, c); break;
        case kGrp: rc = launch_grp(dtype, ldl, c); break;
        case kBlk: rc = launch_blk(dtype, ldl, c); break;
        case kLane: rc = launch_lane(dtype, ldl, c); break;
        case kGeneric: break;
    }
    if (rc == kNoKernel && c.n <= lane_max_n(dtype)) rc = launch_lane(dtype, ldl, c);   // k_grp declined
    if (rc == kNoKernel) rc = launch_generic(dtype, ldl, c);
    return rc;
}

// vectors: interleaved (sm = 1, se >= batch) or contiguous (se = 1, sm >= n)
bool vec_ok(int64_t batch, int n, int64_t sm, int64_t se) {
    if (sm < 1 || se < 1) return false;
    if (n == 1) return true;
    return (sm == 1 && se >= batch) || (se == 1 && sm >= n);
}

int run_solve(int dtype, bool ldl, const SolveArgs& c) {
    const size_t eb = dtype == 0 ? 8 : 16;
    if (c.batch < 0) return -1;
    if (c.n < 1 || c.n > HPDINV_MAX_N) return -2;
    if (c.batch == 0) return 0;
    if (!c.A || reinterpret_cast<uintptr_t>(c.A) % eb) return -3;
    if (classify(c.batch, c.n, c.sAm, c.sAe) == kInvalid) return -4;
    if (!c.Y || reinterpret_cast<uintptr_t>(c.Y) % eb) return -6;
    if (!vec_ok(c.batch, c.n, c.sYm, c.sYe)) return -7;
    if (!c.X || reinterpret_cast<uintptr_t>(c.X) % eb) return -9;
    if (!vec_ok(c.batch, c.n, c.sXm, c.sXe)) return -10;
    if (!c.info || reinterpret_cast<uintptr_t>(c.info) % 4) return -12;
    return launch_solve(dtype, ldl, c);
}

}  // namespace

extern "C" {

int chol_solve_batched_c64(int64_t batch, int n, const cuFloatComplex* A, int64_t sAm, int64_t sAe,
                           const cuFloatComplex* Y, int64_t sYm, int64_t sYe,
                           cuFloatComplex* Xv, int64_t sXm, int64_t sXe, int32_t* info, cudaStream_t stream) {
    return run_solve(0, false, SolveArgs{batch, n, A, sAm, sAe, Y, sYm, sYe, Xv, sXm, sXe, info, stream});
}

int chol_solve_batched_c128(int64_t batch, int n, const cuDoubleComplex* A, int64_t sAm, int64_t sAe,
                            const cuDoubleComplex* Y, int64_t sYm, int64_t sYe,
                            cuDoubleComplex* Xv, int64_t sXm, int64_t sXe, int32_t* info, cudaStream_t stream) {
    return run_solve(1, false, SolveArgs{batch, n, A, sAm, sAe, Y, sYm, sYe, Xv, sXm, sXe, info, stream});
}

int ldl_solve_batched_c64(int64_t batch, int n, const cuFloatComplex* A, int64_t sAm, int64_t sAe,
                          const cuFloatComplex* Y, int64_t sYm, int64_t sYe,
                          cuFloatComplex* Xv, int64_t sXm, int64_t sXe, int32_t* info, cudaStream_t stream) {
    return run_solve(0, true, SolveArgs{batch, n, A, sAm, sAe, Y, sYm, sYe, Xv, sXm, sXe, info, stream});
}

int ldl_solve_batched_c128(int64_t batch, int n, const cuDoubleComplex* A, int64_t sAm, int64_t sAe,
                           const cuDoubleComplex* Y, int64_t sYm, int64_t sYe,
                           cuDoubleComplex* Xv, int64_t sXm, int64_t sXe, int32_t* info, cudaStream_t stream) {
    return run_solve(1, true, SolveArgs{batch, n, A, sAm, sAe, Y, sYm, sYe, Xv, sXm, sXe, info, stream});
}

int hpdinv_inv_batched_method(int method, int dtype, int64_t batch, int n, const void* A, int64_t sAm,
                              int64_t sAe, void* X, int64_t sXm, int64_t sXe, int32_t* info,
                              cudaStream_t stream) {
    if (dtype < 0 || dtype > 1) return -2;
    if (method < 0 || method > 3) return -1;
    const LaunchArgs c{batch, n, A, sAm, sAe, X, sXm, sXe, info, stream};
    int rc;
    if (method <= 1) {
        rc = run(dtype, method == 1, c);
    } else {
        const int v = validate(c, dtype == 0 ? 8 : 16);
        rc = v <= 0 ? v : launch_base(method, dtype, c);
    }
    return (rc < 0 && rc > kNoKernel) ? rc - 2 : rc;   // argument k of the 10-argument form is k+2 here
}

int nonherm_inv_batched_c64(int64_t batch, int n, const cuFloatComplex* D, int64_t sDm, int64_t sDe,
                            cuFloatComplex* Dinv, int64_t sXm, int64_t sXe, int32_t* info, cudaStream_t stream) {
    const LaunchArgs c{batch, n, D, sDm, sDe, Dinv, sXm, sXe, info, stream};
    const int v = validate(c, 8);
    return v <= 0 ? v : launch_nh(0, c);
}

int nonherm_inv_batched_c128(int64_t batch, int n, const cuDoubleComplex* D, int64_t sDm, int64_t sDe,
                             cuDoubleComplex* Dinv, int64_t sXm, int64_t sXe, int32_t* info, cudaStream_t stream) {
    const LaunchArgs c{batch, n, D, sDm, sDe, Dinv, sXm, sXe, info, stream};
    const int v = validate(c, 16);
    return v <= 0 ? v : launch_nh(1, c);
}

const char* hpdinv_nonherm_kernel_name(int dtype, int n) {
    if (n < 1 || n > HPDINV_MAX_N || dtype < 0 || dtype > 1) return nullptr;
    return nh_kernel_name(dtype, n);
}

const char* hpdinv_method_kernel_name(int method, int dtype, int n) {
    if (n < 1 || n > HPDINV_MAX_N || dtype < 0 || dtype > 1) return nullptr;
    return base_kernel_name(method, dtype, n);
}

const char* hpdinv_solve_kernel_name(int method, int dtype, int n) {
    if (n < 1 || n > HPDINV_MAX_N || dtype < 0 || dtype > 1) return nullptr;
    return solve_kernel_name(dtype, method != 0, n);
}


int chol_inv_batched_c64(int64_t batch, int n, const cuFloatComplex* A, int64_t sAm, int64_t sAe,
                         cuFloatComplex* X, int64_t sXm, int64_t sXe, int32_t* info,
                         cudaStream_t stream) {
    return run(0, false, LaunchArgs{batch, n, A, sAm, sAe, X, sXm, sXe, info, stream});
}

int chol_inv_batched_c128(int64_t batch, int n, const cuDoubleComplex* A, int64_t sAm, int64_t sAe,
                          cuDoubleComplex* X, int64_t sXm, int64_t sXe, int32_t* info,
                          cudaStream_t stream) {
    return run(1, false, LaunchArgs{batch, n, A, sAm, sAe, X, sXm, sXe, info, stream});
}

int ldl_inv_batched_c64(int64_t batch, int n, const cuFloatComplex* A, int64_t sAm, int64_t sAe,
                        cuFloatComplex* X, int64_t sXm, int64_t sXe, int32_t* info,
                        cudaStream_t stream) {
    return run(0, true, LaunchArgs{batch, n, A, sAm, sAe, X, sXm, sXe, info, stream});
}

int ldl_inv_batched_c128(int64_t batch, int n, const cuDoubleComplex* A, int64_t sAm, int64_t sAe,
                         cuDoubleComplex* X, int64_t sXm, int64_t sXe, int32_t* info,
                         cudaStream_t stream) {
    return run(1, true, LaunchArgs{batch, n, A, sAm, sAe, X, sXm, sXe, info, stream});
}

const char* hpdinv_kernel_name(int method, int dtype, int64_t batch, int n, int64_t sAm,
                               int64_t sAe, int64_t sXm, int64_t sXe) {
    if (batch < 0 || n < 1 || n > HPDINV_MAX_N || dtype < 0 || dtype > 1) return nullptr;
    if (classify(batch, n, sAm, sAe) == kInvalid || classify(batch, n, sXm, sXe) == kInvalid)
        return nullptr;
    const bool soa = classify(batch, n, sAm, sAe) == kSoA && classify(batch, n, sXm, sXe) == kSoA;
    Family f = family(dtype, n, soa);
    // the same decision launch_grp takes (it declines plane strides >= 4 GiB -> k_lane)
    if (f == kGrp && !grp_strides_ok(sAe, sXe, dtype == 0 ? 8 : 16)) f = n <= lane_max_n(dtype) ? kLane : kGeneric;
    if (classify(batch, n, sAm, sAe) == kAoS && dmma_accepts(dtype, method != 0, n, sAm, sAe)) return "k_dmma<c128,chol>";
    return family_name(f, dtype, method != 0);
}

const char* hpdinv_version(void) { return "hpdinv 0.2.0 (sm_100a)"; }

}  // extern "C"
