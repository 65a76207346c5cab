// cplx.cuh -- complex scalar helpers for the device kernels (fp32 / fp64).
// Part of the product path; independent of oracle/ (no shared code).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hpdinv {

template <typename T> struct vec2;
template <> struct vec2<float> { using type = float2; };
template <> struct vec2<double> { using type = double2; };
template <typename T> using cplx = typename vec2<T>::type;

template <typename T> __device__ __forceinline__ cplx<T> mk(T re, T im) { cplx<T> z; z.x = re; z.y = im; return z; }
template <typename T> __device__ __forceinline__ cplx<T> czero() { return mk<T>(T(0), T(0)); }

template <typename T> __device__ __forceinline__ T qnan();
template <> __device__ __forceinline__ float qnan<float>() { return __int_as_float(0x7fc00000); }
template <> __device__ __forceinline__ double qnan<double>() { return __longlong_as_double(0x7ff8000000000000ULL); }

// Overloads (not templates: cplx<T> is a non-deduced context).
#define HPDINV_CPLX_COMMON(V, T)                                                                   \
    __device__ __forceinline__ V conjz(V a) { V z; z.x = a.x; z.y = -a.y; return z; }              \
    /* acc += a * conj(b) */                                                                       \
    __device__ __forceinline__ void cfma_conjb(V& acc, V a, V b) {                                 \
        acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);                                \
        acc.y = fma(a.y, b.x, acc.y); acc.y = fma(-a.x, b.y, acc.y); }                             \
    /* t + Re(a * conj(b)) */                                                                      \
    __device__ __forceinline__ T re_dot_conj(T t, V a, V b) { t = fma(a.x, b.x, t); return fma(a.y, b.y, t); } \
    __device__ __forceinline__ V cscale(V a, T s) { V z; z.x = a.x * s; z.y = a.y * s; return z; }

#define HPDINV_CPLX_SCALAR_MAC(V)                                                                  \
    /* acc += a * b */                                                                             \
    __device__ __forceinline__ void cfma(V& acc, V a, V b) {                                       \
        acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);                               \
        acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y); }                              \
    /* acc -= a * b */                                                                             \
    __device__ __forceinline__ void cfms(V& acc, V a, V b) {                                       \
        acc.x = fma(-a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);                               \
        acc.y = fma(-a.x, b.y, acc.y); acc.y = fma(-a.y, b.x, acc.y); }                            \
    /* acc -= conj(a) * b */                                                                       \
    __device__ __forceinline__ void cfms_conj(V& acc, V a, V b) {                                  \
        acc.x = fma(-a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);                              \
        acc.y = fma(-a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y); }

HPDINV_CPLX_COMMON(double2, double)
HPDINV_CPLX_SCALAR_MAC(double2)
HPDINV_CPLX_COMMON(float2, float)

#ifdef HPDINV_NO_FFMA2
HPDINV_CPLX_SCALAR_MAC(float2)
#else
// fp32 complex multiply-accumulate on the packed FFMA2 path of sm_100a: one complex MAC is two
// fma.rn.f32x2 with the per-element operand b broadcast as a scalar ((b.re, b.re), (b.im, b.im))
// and the operand a (the one the kernels share across a lane's columns: an R element read by
// broadcast) arranged as a pair.  ptxas folds the scalar broadcasts, the swap and the negation
// into FFMA2 operand modifiers (.F32, .LO_HI, -), so a MAC issues two instructions (plus one
// FADD per shared a for the conjugated forms).  Every lane is one IEEE fma:
//   cfma:      re' = fma(b.im, -a.im, fma(b.re, a.re, re)),  im' = fma(b.im, a.re, fma(b.re, a.im, im))
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(unsigned long long v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
// acc += a * b
__device__ __forceinline__ void cfma(float2& acc, float2 a, float2 b) {
    unsigned long long c = pk2(acc.x, acc.y);
    c = ffma2(pk2(b.x, b.x), pk2(a.x, a.y), c);
    c = ffma2(pk2(b.y, b.y), pk2(-a.y, a.x), c);
    upk2(c, acc.x, acc.y);
}
// acc -= a * b
__device__ __forceinline__ void cfms(float2& acc, float2 a, float2 b) {
    unsigned long long c = pk2(acc.x, acc.y);
    c = ffma2(pk2(b.x, b.x), pk2(-a.x, -a.y), c);
    c = ffma2(pk2(b.y, b.y), pk2(a.y, -a.x), c);
    upk2(c, acc.x, acc.y);
}
// acc -= conj(a) * b
__device__ __forceinline__ void cfms_conj(float2& acc, float2 a, float2 b) {
    unsigned long long c = pk2(acc.x, acc.y);
    c = ffma2(pk2(b.x, b.x), pk2(-a.x, a.y), c);
    c = ffma2(pk2(b.y, b.y), pk2(-a.y, -a.x), c);
    upk2(c, acc.x, acc.y);
}
#endif
#undef HPDINV_CPLX_COMMON
#undef HPDINV_CPLX_SCALAR_MAC

// IEEE round-to-nearest reciprocal and square root (exact at 1.0; R9).
__device__ __forceinline__ float rcp_rn(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp_rn(double x) { return __drcp_rn(x); }
__device__ __forceinline__ float sqrt_rn(float x) { return __fsqrt_rn(x); }
__device__ __forceinline__ double sqrt_rn(double x) { return __dsqrt_rn(x); }

// Packed upper-triangle index, row-major: (i, j), i <= j, of an n x n matrix.
__host__ __device__ constexpr int upk(int n, int i, int j) { return i * n - (i * (i - 1)) / 2 + (j - i); }

}  // namespace hpdinv
