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
#define HPDINV_CPLX_OPS(V, T)                                                                      \
    __device__ __forceinline__ V conjz(V a) { V z; z.x = a.x; z.y = -a.y; return z; }              \
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
        acc.y = fma(-a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y); }                             \
    /* acc += a * conj(b) */                                                                       \
    __device__ __forceinline__ void cfma_conjb(V& acc, V a, V b) {                                 \
        acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);                                \
        acc.y = fma(a.y, b.x, acc.y); acc.y = fma(-a.x, b.y, acc.y); }                             \
    /* t + Re(a * conj(b)) */                                                                      \
    __device__ __forceinline__ T re_dot_conj(T t, V a, V b) { t = fma(a.x, b.x, t); return fma(a.y, b.y, t); } \
    __device__ __forceinline__ V cscale(V a, T s) { V z; z.x = a.x * s; z.y = a.y * s; return z; }

HPDINV_CPLX_OPS(float2, float)
HPDINV_CPLX_OPS(double2, double)
#undef HPDINV_CPLX_OPS

// IEEE round-to-nearest reciprocal and square root (exact at 1.0; R9).
__device__ __forceinline__ float rcp_rn(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp_rn(double x) { return __drcp_rn(x); }
__device__ __forceinline__ float sqrt_rn(float x) { return __fsqrt_rn(x); }
__device__ __forceinline__ double sqrt_rn(double x) { return __dsqrt_rn(x); }

// Packed upper-triangle index, row-major: (i, j), i <= j, of an n x n matrix.
__host__ __device__ constexpr int upk(int n, int i, int j) { return i * n - (i * (i - 1)) / 2 + (j - i); }

}  // namespace hpdinv
