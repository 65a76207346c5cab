// peaks.cu -- FP32 (FFMA, FFMA2) and FP64 (DFMA) issue-rate microbenchmark for the roofline
// denominators of the compute-bound configs.  Each thread runs 8 independent
// FMA chains; the grid is 148 x 8 CTAs of 256 threads.  Prints TFLOP/s (2 flops per FMA).
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
    T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 16; u++) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void ffma2_loop(float* out, int iters, float a, float b) {
    unsigned long long x[8], va, vb;
    float2 fa = make_float2(a, a), fb = make_float2(b, b);
    va = *reinterpret_cast<unsigned long long*>(&fa);
    vb = *reinterpret_cast<unsigned long long*>(&fb);
    for (int k = 0; k < 8; k++) { float2 f = make_float2(threadIdx.x + k, k); x[k] = *reinterpret_cast<unsigned long long*>(&f); }
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 16; u++)
#pragma unroll
            for (int k = 0; k < 8; k++)
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[k]) : "l"(va), "l"(vb));
    }
    float s = 0;
    for (int k = 0; k < 8; k++) { float2 f = *reinterpret_cast<float2*>(&x[k]); s += f.x + f.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float time_it(F f) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); cudaDeviceSynchronize();
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}

int main() {
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    void* out; cudaMalloc(&out, blocks * threads * 8);
    double fmas = double(blocks) * threads * iters * 16 * 8;
    float ms = time_it([&] { fma_loop<float><<<blocks, threads>>>((float*)out, iters, 0.999f, 0.001f); });
    printf("{\"ffma_tflops\": %.2f, ", 2 * fmas / ms / 1e9);
    ms = time_it([&] { ffma2_loop<<<blocks, threads>>>((float*)out, iters, 0.999f, 0.001f); });
    printf("\"ffma2_tflops\": %.2f, ", 2 * 2 * fmas / ms / 1e9);
    ms = time_it([&] { fma_loop<double><<<blocks, threads>>>((double*)out, iters / 4, 0.999, 0.001); });
    printf("\"dfma_tflops\": %.2f}\n", 2 * fmas / 4 / ms / 1e9);
    return 0;
}
