// api.cu -- the C ABI of include/hpdinv.h: argument validation, layout classification,
// kernel selection per (method, dtype, n, layout) and the launch.  Host code only; the
// kernels live in the k_*.cuh headers.
#include <cstdio>
#include <mutex>
#include <set>
#include <utility>

#include "../../include/hpdinv.h"
#include "cplx.cuh"
#include "k_generic.cuh"
#include "k_reg.cuh"

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

// Raise the dynamic shared-memory limit of `fn` on the current device once.
cudaError_t ensure_smem(const void* fn, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({fn, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    if (e == cudaSuccess) done.insert({fn, dev});
    return e;
}

struct Call {
    int method;  // 0 Cholesky, 1 LDL
    int64_t batch;
    int n;
    const void* A;
    int64_t sAm, sAe;
    void* X;
    int64_t sXm, sXe;
    int32_t* info;
    cudaStream_t stream;
};

// ------------------------------------------------------------------ kernel table
template <typename T, bool LDL>
struct Family {
    using reg_fn = void (*)(int64_t, const cplx<T>*, int64_t, int64_t, cplx<T>*, int64_t, int64_t,
                            int32_t*);
    static constexpr int kMaxReg = sizeof(T) == 4 ? 8 : 6;

    static reg_fn reg_kernel(int n) {
        switch (n) {
            case 1: return k_reg<T, 1, LDL>;
            case 2: return k_reg<T, 2, LDL>;
            case 3: return k_reg<T, 3, LDL>;
            case 4: return k_reg<T, 4, LDL>;
            case 5: return k_reg<T, 5, LDL>;
            case 6: return k_reg<T, 6, LDL>;
#define HPDINV_REG_BIG(NN) case NN: return sizeof(T) == 4 ? reg_fn(k_reg<T, NN, LDL>) : nullptr;
            HPDINV_REG_BIG(7)
            HPDINV_REG_BIG(8)
#undef HPDINV_REG_BIG
            default: return nullptr;
        }
    }

    static const char* name(int n, bool* use_reg) {
        *use_reg = n <= kMaxReg;
        return *use_reg ? (sizeof(T) == 4 ? (LDL ? "k_reg<c64,ldl>" : "k_reg<c64,chol>")
                                          : (LDL ? "k_reg<c128,ldl>" : "k_reg<c128,chol>"))
                        : (sizeof(T) == 4 ? (LDL ? "k_generic<c64,ldl>" : "k_generic<c64,chol>")
                                          : (LDL ? "k_generic<c128,ldl>" : "k_generic<c128,chol>"));
    }

    static int launch(const Call& c) {
        const cplx<T>* A = static_cast<const cplx<T>*>(c.A);
        cplx<T>* X = static_cast<cplx<T>*>(c.X);
        if (c.n <= kMaxReg) {
            reg_fn fn = reg_kernel(c.n);
            const int64_t blocks = (c.batch + kRegThreads - 1) / kRegThreads;
            fn<<<unsigned(blocks), kRegThreads, 0, c.stream>>>(c.batch, A, c.sAm, c.sAe, X, c.sXm,
                                                               c.sXe, c.info);
        } else {
            const size_t smem = generic_smem_bytes<T>(c.n);
            auto fn = k_generic<T, LDL>;
            cudaError_t e = ensure_smem(reinterpret_cast<const void*>(fn), smem);
            if (e != cudaSuccess) return int(e);
            const int64_t blocks = c.batch < (int64_t(1) << 30) ? c.batch : (int64_t(1) << 30);
            fn<<<unsigned(blocks), kGenericThreads, smem, c.stream>>>(c.batch, c.n, A, c.sAm, c.sAe,
                                                                     X, c.sXm, c.sXe, c.info);
        }
        return int(cudaGetLastError());
    }
};

int validate(const Call& c, size_t elem_bytes) {
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

template <typename T>
int run(const Call& c) {
    int v = validate(c, sizeof(cplx<T>));
    if (v <= 0) return v;
    return c.method == 1 ? Family<T, true>::launch(c) : Family<T, false>::launch(c);
}

}  // namespace

extern "C" {

int chol_inv_batched_c64(int64_t batch, int n, const cuFloatComplex* A, int64_t sAm, int64_t sAe,
                         cuFloatComplex* X, int64_t sXm, int64_t sXe, int32_t* info,
                         cudaStream_t stream) {
    return run<float>(Call{0, batch, n, A, sAm, sAe, X, sXm, sXe, info, stream});
}

int chol_inv_batched_c128(int64_t batch, int n, const cuDoubleComplex* A, int64_t sAm, int64_t sAe,
                          cuDoubleComplex* X, int64_t sXm, int64_t sXe, int32_t* info,
                          cudaStream_t stream) {
    return run<double>(Call{0, batch, n, A, sAm, sAe, X, sXm, sXe, info, stream});
}

int ldl_inv_batched_c64(int64_t batch, int n, const cuFloatComplex* A, int64_t sAm, int64_t sAe,
                        cuFloatComplex* X, int64_t sXm, int64_t sXe, int32_t* info,
                        cudaStream_t stream) {
    return run<float>(Call{1, batch, n, A, sAm, sAe, X, sXm, sXe, info, stream});
}

int ldl_inv_batched_c128(int64_t batch, int n, const cuDoubleComplex* A, int64_t sAm, int64_t sAe,
                         cuDoubleComplex* X, int64_t sXm, int64_t sXe, int32_t* info,
                         cudaStream_t stream) {
    return run<double>(Call{1, batch, n, A, sAm, sAe, X, sXm, sXe, info, stream});
}

const char* hpdinv_kernel_name(int method, int dtype, int64_t batch, int n, int64_t sAm,
                               int64_t sAe, int64_t sXm, int64_t sXe) {
    if (batch < 0 || n < 1 || n > HPDINV_MAX_N) return nullptr;
    if (classify(batch, n, sAm, sAe) == kInvalid || classify(batch, n, sXm, sXe) == kInvalid)
        return nullptr;
    bool reg;
    if (dtype == 0) return method ? Family<float, true>::name(n, &reg) : Family<float, false>::name(n, &reg);
    return method ? Family<double, true>::name(n, &reg) : Family<double, false>::name(n, &reg);
}

const char* hpdinv_version(void) { return "hpdinv 0.1.0 (sm_100a)"; }

}  // extern "C"
