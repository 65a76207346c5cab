// mma_peaks.cu -- tensor-core (mma.sync) throughput on sm_100a for the FP64 and TF32 shapes
// the blocked kernels could use, next to the DFMA pipe:
//   dmma_m8n8k4    mma.sync.aligned.m8n8k4.row.col.f64       (256 FMA per warp instruction)
//   dmma_m16n8k4   mma.sync.aligned.m16n8k4.row.col.f64      (512)
//   dmma_m16n8k8   mma.sync.aligned.m16n8k8.row.col.f64      (1024)
//   dmma_m16n8k16  mma.sync.aligned.m16n8k16.row.col.f64     (2048)
//   tf32_m16n8k8   mma.sync.aligned.m16n8k8.row.col.f32.tf32 (1024)
//   dfma           plain DFMA, 8 independent chains
//   mix            half the warps DMMA m8n8k4, half DFMA (do the two share a pipe?)
// Grid 148 x WPB/... CTAs, 8 independent accumulators per warp.  Prints TFLOP/s (2 flops/FMA).
#include <cstdio>
#include <cuda_runtime.h>

#define ACC 8

__device__ __forceinline__ void mma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1684(double (&d)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void mma1688(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
__device__ __forceinline__ void tf32_1688(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__global__ void k884(double* out, int iters, const double* seed) {
    double d[ACC][2] = {};
    double a = seed[threadIdx.x & 63], b = seed[(threadIdx.x + 5) & 63];
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < ACC; k++) mma884(d[k], a, b);
    double s = 0;
    for (int k = 0; k < ACC; k++) s += d[k][0] + d[k][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k1684(double* out, int iters, const double* seed) {
    double d[ACC][4] = {};
    double a0 = seed[threadIdx.x & 63], a1 = seed[(threadIdx.x + 3) & 63], b = seed[(threadIdx.x + 5) & 63];
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < ACC; k++) mma1684(d[k], a0, a1, b);
    double s = 0;
    for (int k = 0; k < ACC; k++) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k1688(double* out, int iters, const double* seed) {
    double d[ACC][4] = {};
    double a[4], b[2];
    for (int k = 0; k < 4; k++) a[k] = seed[(threadIdx.x + k) & 63];
    for (int k = 0; k < 2; k++) b[k] = seed[(threadIdx.x + 7 + k) & 63];
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < ACC; k++) mma1688(d[k], a, b);
    double s = 0;
    for (int k = 0; k < ACC; k++) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k16816(double* out, int iters, const double* seed) {
    double d[ACC][4] = {};
    double a[8], b[4];
    for (int k = 0; k < 8; k++) a[k] = seed[(threadIdx.x + k) & 63];
    for (int k = 0; k < 4; k++) b[k] = seed[(threadIdx.x + 7 + k) & 63];
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < ACC; k++) mma16816(d[k], a, b);
    double s = 0;
    for (int k = 0; k < ACC; k++) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ktf32(float* out, int iters, const float* seed) {
    float d[ACC][4] = {};
    unsigned a[4], b[2];
    for (int k = 0; k < 4; k++) a[k] = __float_as_uint(seed[(threadIdx.x + k) & 63]);
    for (int k = 0; k < 2; k++) b[k] = __float_as_uint(seed[(threadIdx.x + 7 + k) & 63]);
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < ACC; k++) tf32_1688(d[k], a, b);
    float s = 0;
    for (int k = 0; k < ACC; k++) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void kdfma(double* out, int iters, double a, double b) {
    double x[ACC];
    for (int k = 0; k < ACC; k++) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int u = 0; u < 8; u++)
#pragma unroll
            for (int k = 0; k < ACC; k++) x[k] = fma(x[k], a, b);
    double s = 0;
    for (int k = 0; k < ACC; k++) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// even warps: DMMA m8n8k4 (iters_m), odd warps: DFMA (iters_f)
__global__ void kmix(double* out, int iters_m, int iters_f, const double* seed) {
    double s = 0;
    if ((threadIdx.x >> 5) & 1) {
        double x[ACC];
        for (int k = 0; k < ACC; k++) x[k] = threadIdx.x + k;
        const double a = seed[1], b = seed[2];
        for (int i = 0; i < iters_f; i++)
#pragma unroll
            for (int u = 0; u < 8; u++)
#pragma unroll
                for (int k = 0; k < ACC; k++) x[k] = fma(x[k], a, b);
        for (int k = 0; k < ACC; k++) s += x[k];
    } else {
        double d[ACC][2] = {};
        double a = seed[threadIdx.x & 63], b = seed[(threadIdx.x + 5) & 63];
        for (int i = 0; i < iters_m; i++)
#pragma unroll
            for (int k = 0; k < ACC; k++) mma884(d[k], a, b);
        for (int k = 0; k < ACC; k++) s += d[k][0] + d[k][1];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float time_it(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; r++) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    const int threads = 256, blocks = 148 * 4;
    void* out;
    cudaMalloc(&out, size_t(blocks) * threads * 8);
    double hs[64];
    for (int i = 0; i < 64; i++) hs[i] = 1e-3 * (i % 7) - 2e-3;
    void* seed;
    cudaMalloc(&seed, 64 * 8);
    cudaMemcpy(seed, hs, sizeof(hs), cudaMemcpyHostToDevice);
    float hf[64];
    for (int i = 0; i < 64; i++) hf[i] = float(hs[i]);
    void* seedf;
    cudaMalloc(&seedf, 64 * 4);
    cudaMemcpy(seedf, hf, sizeof(hf), cudaMemcpyHostToDevice);
    const double warps = double(blocks) * threads / 32;
    const int it = 2048;
    float ms;
    ms = time_it([&] { k884<<<blocks, threads>>>((double*)out, it, (const double*)seed); });
    printf("{\"dmma_m8n8k4_tflops\": %.2f, ", 2.0 * warps * it * ACC * 256 / ms / 1e9);
    ms = time_it([&] { k1684<<<blocks, threads>>>((double*)out, it, (const double*)seed); });
    printf("\"dmma_m16n8k4_tflops\": %.2f, ", 2.0 * warps * it * ACC * 512 / ms / 1e9);
    ms = time_it([&] { k1688<<<blocks, threads>>>((double*)out, it / 2, (const double*)seed); });
    printf("\"dmma_m16n8k8_tflops\": %.2f, ", 2.0 * warps * (it / 2) * ACC * 1024 / ms / 1e9);
    ms = time_it([&] { k16816<<<blocks, threads>>>((double*)out, it / 4, (const double*)seed); });
    printf("\"dmma_m16n8k16_tflops\": %.2f, ", 2.0 * warps * (it / 4) * ACC * 2048 / ms / 1e9);
    ms = time_it([&] { ktf32<<<blocks, threads>>>((float*)out, it, (const float*)seedf); });
    printf("\"tf32_mma_m16n8k8_tflops\": %.2f, ", 2.0 * warps * it * ACC * 1024 / ms / 1e9);
    ms = time_it([&] { kdfma<<<blocks, threads>>>((double*)out, it / 4, 0.999, 1e-3); });
    const double dfma_tf = 2.0 * blocks * threads * (it / 4) * 8.0 * ACC / ms / 1e9;
    printf("\"dfma_tflops\": %.2f, ", dfma_tf);
    // mix: half the warps each; report the total FP64 rate
    ms = time_it([&] { kmix<<<blocks, threads>>>((double*)out, it / 2, it / 32, (const double*)seed); });
    const double mix_flops = 2.0 * (warps / 2) * (it / 2) * ACC * 256 + 2.0 * (blocks * threads / 2.0) * (it / 32) * 8.0 * ACC;
    printf("\"mix_dmma_dfma_tflops\": %.2f, \"mix_ms\": %.3f}\n", mix_flops / ms / 1e9, ms);
    return 0;
}
