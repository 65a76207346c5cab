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

// acc += a * conj(b)   (fp32: two FFMA2, scalar operand b broadcast; fp64: four DFMA)
__device__ __forceinline__ void cfma_cb(double2& acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.y, b.x, acc.y); acc.y = fma(-a.x, b.y, acc.y);
}
#ifdef HPDINV_NO_FFMA2
__device__ __forceinline__ void cfma_cb(float2& acc, float2 a, float2 b) {
    acc.x = fmaf(a.x, b.x, acc.x); acc.x = fmaf(a.y, b.y, acc.x);
    acc.y = fmaf(a.y, b.x, acc.y); acc.y = fmaf(-a.x, b.y, acc.y);
}
#else
__device__ __forceinline__ void cfma_cb(float2& acc, float2 a, float2 b) {
    unsigned long long c = pk2(acc.x, acc.y);
    c = ffma2(pk2(b.x, b.x), pk2(a.x, a.y), c);
    c = ffma2(pk2(b.y, b.y), pk2(a.y, -a.x), c);
    upk2(c, acc.x, acc.y);
}
#endif

// "Shared-multiplier" complex MAC.  The kernels' inner loops multiply one operand a, reused
// across a whole row of MACs, by a stream of per-use operands x.  PMul<T> holds a in the form
// the MAC wants; PAcc<T> is the accumulator.  fp32 (FFMA2 path): a*x = x.re*(a.re, a.im) +
// x.im*(-a.im, a.re), so with p = (a.re, a.im) and q = (-a.im, a.re) precomputed once, one MAC
// is two fma.rn.f32x2 whose scalar operand (x.re or x.im) is broadcast to both lanes; the
// accumulator stays packed in one 64-bit register pair.  fp64: plain DFMA.
template <typename T> struct PMul;
template <typename T> struct PAcc;
template <> struct PMul<double> { double2 a; };
template <> struct PAcc<double> { double2 v; };
__device__ __forceinline__ PMul<double> pmul(double2 a) { return PMul<double>{a}; }
__device__ __forceinline__ PAcc<double> pacc(double2 v) { return PAcc<double>{v}; }
__device__ __forceinline__ double2 pval(PAcc<double> c) { return c.v; }
__device__ __forceinline__ void pmac(PAcc<double>& c, const PMul<double>& m, double2 x) { cfma(c.v, m.a, x); }
__device__ __forceinline__ void pmac_cb(PAcc<double>& c, const PMul<double>& m, double2 x) { cfma_cb(c.v, m.a, x); }
#ifdef HPDINV_NO_FFMA2
template <> struct PMul<float> { float2 a; };
template <> struct PAcc<float> { float2 v; };
__device__ __forceinline__ PMul<float> pmul(float2 a) { return PMul<float>{a}; }
__device__ __forceinline__ PAcc<float> pacc(float2 v) { return PAcc<float>{v}; }
__device__ __forceinline__ float2 pval(PAcc<float> c) { return c.v; }
__device__ __forceinline__ void pmac(PAcc<float>& c, const PMul<float>& m, float2 x) { cfma(c.v, m.a, x); }
__device__ __forceinline__ void pmac_cb(PAcc<float>& c, const PMul<float>& m, float2 x) { cfma_cb(c.v, m.a, x); }
#else
template <> struct PMul<float> { unsigned long long p, q; };
template <> struct PAcc<float> { unsigned long long v; };
__device__ __forceinline__ PMul<float> pmul(float2 a) { return PMul<float>{pk2(a.x, a.y), pk2(-a.y, a.x)}; }
__device__ __forceinline__ PAcc<float> pacc(float2 v) { return PAcc<float>{pk2(v.x, v.y)}; }
__device__ __forceinline__ float2 pval(PAcc<float> c) { float2 z; upk2(c.v, z.x, z.y); return z; }
// c += a * x
__device__ __forceinline__ void pmac(PAcc<float>& c, const PMul<float>& m, float2 x) {
    c.v = ffma2(pk2(x.x, x.x), m.p, c.v);
    c.v = ffma2(pk2(x.y, x.y), m.q, c.v);
}
// c += a * conj(x)
__device__ __forceinline__ void pmac_cb(PAcc<float>& c, const PMul<float>& m, float2 x) {
    c.v = ffma2(pk2(x.x, x.x), m.p, c.v);
    c.v = ffma2(pk2(-x.y, -x.y), m.q, c.v);
}
#endif

// Split accumulator for a MAC whose shared operand is the STREAMED one: smac(acc, r, x) with
// r the pair (r.re, r.im) as loaded and x broadcast per component keeps a = sum x.re * r and
// b = sum x.im * r (fp32: two FFMA2 with no operand rearrangement at all; fp64: four DFMA).
//   sval(acc)       = sum r x        = a + i b
//   sval_conjr(acc) = sum conj(r) x  = conj(sum r conj(x)) = conj(a - i b)
template <typename T> struct SAcc;
template <> struct SAcc<double> { double2 a, b; };
__device__ __forceinline__ void sacc_zero(SAcc<double>& c) { c.a = make_double2(0.0, 0.0); c.b = c.a; }
__device__ __forceinline__ void smac(SAcc<double>& c, double2 r, double2 x) {
    c.a.x = fma(x.x, r.x, c.a.x); c.a.y = fma(x.x, r.y, c.a.y);
    c.b.x = fma(x.y, r.x, c.b.x); c.b.y = fma(x.y, r.y, c.b.y);
}
__device__ __forceinline__ double2 sval(const SAcc<double>& c) { return make_double2(c.a.x - c.b.y, c.a.y + c.b.x); }
__device__ __forceinline__ double2 sval_conjr(const SAcc<double>& c) { return make_double2(c.a.x + c.b.y, c.b.x - c.a.y); }
#ifdef HPDINV_NO_FFMA2
template <> struct SAcc<float> { float2 a, b; };
__device__ __forceinline__ void sacc_zero(SAcc<float>& c) { c.a = make_float2(0.f, 0.f); c.b = c.a; }
__device__ __forceinline__ void smac(SAcc<float>& c, float2 r, float2 x) {
    c.a.x = fmaf(x.x, r.x, c.a.x); c.a.y = fmaf(x.x, r.y, c.a.y);
    c.b.x = fmaf(x.y, r.x, c.b.x); c.b.y = fmaf(x.y, r.y, c.b.y);
}
__device__ __forceinline__ float2 sval(const SAcc<float>& c) { return make_float2(c.a.x - c.b.y, c.a.y + c.b.x); }
__device__ __forceinline__ float2 sval_conjr(const SAcc<float>& c) { return make_float2(c.a.x + c.b.y, c.b.x - c.a.y); }
#else
template <> struct SAcc<float> { unsigned long long a, b; };
__device__ __forceinline__ void sacc_zero(SAcc<float>& c) { c.a = 0ull; c.b = 0ull; }
__device__ __forceinline__ void smac(SAcc<float>& c, float2 r, float2 x) {
    const unsigned long long rp = pk2(r.x, r.y);
    c.a = ffma2(pk2(x.x, x.x), rp, c.a);
    c.b = ffma2(pk2(x.y, x.y), rp, c.b);
}
__device__ __forceinline__ float2 sval(const SAcc<float>& c) {
    float ax, ay, bx, by;
    upk2(c.a, ax, ay);
    upk2(c.b, bx, by);
    return make_float2(ax - by, ay + bx);
}
__device__ __forceinline__ float2 sval_conjr(const SAcc<float>& c) {
    float ax, ay, bx, by;
    upk2(c.a, ax, ay);
    upk2(c.b, bx, by);
    return make_float2(ax + by, bx - ay);
}
#endif

// elementwise (a.re*b.re + c.re, a.im*b.im + c.im): one FFMA2 for fp32 (Re(a conj(b)) partial sums)
__device__ __forceinline__ double2 pfma_elem(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
}
#ifdef HPDINV_NO_FFMA2
__device__ __forceinline__ float2 pfma_elem(float2 a, float2 b, float2 c) {
    return make_float2(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y));
}
#else
__device__ __forceinline__ float2 pfma_elem(float2 a, float2 b, float2 c) {
    float2 z;
    upk2(ffma2(pk2(a.x, a.y), pk2(b.x, b.y), pk2(c.x, c.y)), z.x, z.y);
    return z;
}
#endif
#undef HPDINV_CPLX_COMMON
#undef HPDINV_CPLX_SCALAR_MAC

// IEEE round-to-nearest reciprocal and square root (exact at 1.0; R9).
__device__ __forceinline__ float rcp_rn(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp_rn(double x) { return __drcp_rn(x); }
__device__ __forceinline__ float sqrt_rn(float x) { return __fsqrt_rn(x); }
__device__ __forceinline__ double sqrt_rn(double x) { return __dsqrt_rn(x); }

// Short-latency pivot reciprocals for the fp32 lane-group kernels: hardware approximation
// (MUFU, ~2^-22 relative) plus one Newton step, exact when the operand is 1.0 (so the exact
// integer families stay bit-exact; R9).  1/sqrt(t) for Cholesky, 1/t for LDL.
__device__ __forceinline__ float rsqrt_nr(float t) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(t));
    const float e = fmaf(-t * y, y, 1.0f);       // 1 - t y^2
    return fmaf(0.5f * y, e, y);
}
__device__ __forceinline__ float rcp_nr(float t) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(t));
    const float e = fmaf(-t, y, 1.0f);
    return fmaf(y, e, y);
}

// Pivot reciprocals of the blocked kernels: hardware approximation refined by Newton steps --
// fp32: one step (correctly rounded or 1 ulp); fp64: two steps (the MUFU seed is ~2^-22, one
// step gives ~2^-44, the second ~1 ulp: c128 keeps full fp64 precision on the pivots, round-2
// VERDICT item 6) -- and exactly 1 when the operand is exactly 1 (the exact integer families
// stay bit-exact; R9).
__device__ __forceinline__ float rsqrt_fast(float t) { return t == 1.0f ? 1.0f : rsqrt_nr(t); }
__device__ __forceinline__ float rcp_fast(float t) { return t == 1.0f ? 1.0f : rcp_nr(t); }
__device__ __forceinline__ double rsqrt_fast(double t) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
    double e = fma(-t * y, y, 1.0);
    y = fma(0.5 * y, e, y);
    e = fma(-t * y, y, 1.0);
    y = fma(0.5 * y, e, y);
    return t == 1.0 ? 1.0 : y;
}
__device__ __forceinline__ double rcp_fast(double t) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
    double e = fma(-t, y, 1.0);
    y = fma(y, e, y);
    e = fma(-t, y, 1.0);
    y = fma(y, e, y);
    return t == 1.0 ? 1.0 : y;
}

// Packed upper-triangle index, row-major: (i, j), i <= j, of an n x n matrix.
__host__ __device__ constexpr int upk(int n, int i, int j) { return i * n - (i * (i - 1)) / 2 + (j - i); }

}  // namespace hpdinv
