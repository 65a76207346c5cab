// peaks.cu -- FP32 (FFMA, FFMA2) and FP64 (DFMA) throughput microbenchmark for the roofline
// denominators of the compute-bound paths.  Variants:
//   *_const : x = fma(x, a, b) with a, b uniform (constant-bank operands)
//   *_reg   : complex multiply-accumulate acc += p * q with every operand in registers
//             (the operand pattern of the kernels' inner loops)
// Grid 148 x 8 CTAs of 256 threads.  Prints TFLOP/s (2 flops per FMA).
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void fma_const(T* out, int iters, T a, T b) {
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

// 4 complex accumulators, 4 x-operands, 2 r-operands per step: 32 FMAs / step, all registers.
template <typename T>
__global__ void cmac_reg(T* out, int iters, T* seed) {
    const int t = threadIdx.x;
    T ax[4], ay[4], xx[4], xy[4], rx[2], ry[2];
    for (int k = 0; k < 4; k++) { ax[k] = 0; ay[k] = 0; xx[k] = seed[(t + k) & 63]; xy[k] = seed[(t + k + 7) & 63]; }
    for (int k = 0; k < 2; k++) { rx[k] = seed[(t + 3 * k + 1) & 63]; ry[k] = seed[(t + 5 * k + 2) & 63]; }
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int r = (k + u) & 1;
                ax[k] = fma(rx[r], xx[k], ax[k]); ax[k] = fma(-ry[r], xy[k], ax[k]);
                ay[k] = fma(rx[r], xy[k], ay[k]); ay[k] = fma(ry[r], xx[k], ay[k]);
            }
            rx[0] += T(1e-7); ry[1] -= T(1e-7);
        }
    }
    T s = 0;
    for (int k = 0; k < 4; k++) s += ax[k] + ay[k];
    out[blockIdx.x * blockDim.x + t] = s;
}

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    float2 f = make_float2(a, b);
    return *reinterpret_cast<unsigned long long*>(&f);
}

// Same complex MAC with packed FFMA2: acc(re,im) += (x.re,x.re)*(r.re,r.im) + (x.im,x.im)*(-r.im,r.re)
__global__ void cmac_ffma2(float* out, int iters, float* seed) {
    const int t = threadIdx.x;
    unsigned long long acc[4], xlo[4], xhi[4], r1[2], r2[2];
    for (int k = 0; k < 4; k++) {
        float a = seed[(t + k) & 63], b = seed[(t + k + 7) & 63];
        acc[k] = pk(0.f, 0.f); xlo[k] = pk(a, a); xhi[k] = pk(b, b);
    }
    for (int k = 0; k < 2; k++) {
        float a = seed[(t + 3 * k + 1) & 63], b = seed[(t + 5 * k + 2) & 63];
        r1[k] = pk(a, b); r2[k] = pk(-b, a);
    }
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int r = (k + u) & 1;
                asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[k]) : "l"(xlo[k]), "l"(r1[r]));
                asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[k]) : "l"(xhi[k]), "l"(r2[r]));
            }
        }
    }
    float s = 0;
    for (int k = 0; k < 4; k++) { float2 f = *reinterpret_cast<float2*>(&acc[k]); s += f.x + f.y; }
    out[blockIdx.x * blockDim.x + t] = s;
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
    void* seed; cudaMalloc(&seed, 64 * 8); cudaMemset(seed, 0, 64 * 8);
    const double th = double(blocks) * threads;
    float ms = time_it([&] { fma_const<float><<<blocks, threads>>>((float*)out, iters, 0.999f, 0.001f); });
    printf("{\"ffma_const_tflops\": %.2f, ", 2 * th * iters * 128 / ms / 1e9);
    ms = time_it([&] { cmac_reg<float><<<blocks, threads>>>((float*)out, iters, (float*)seed); });
    printf("\"ffma_reg_cmac_tflops\": %.2f, ", 2 * th * iters * 128 / ms / 1e9);
    ms = time_it([&] { cmac_ffma2<<<blocks, threads>>>((float*)out, iters, (float*)seed); });
    printf("\"ffma2_reg_cmac_tflops\": %.2f, ", 2 * th * iters * 128 / ms / 1e9);
    ms = time_it([&] { fma_const<double><<<blocks, threads>>>((double*)out, iters / 4, 0.999, 0.001); });
    printf("\"dfma_const_tflops\": %.2f, ", 2 * th * iters / 4 * 128 / ms / 1e9);
    ms = time_it([&] { cmac_reg<double><<<blocks, threads>>>((double*)out, iters / 4, (double*)seed); });
    printf("\"dfma_reg_cmac_tflops\": %.2f}\n", 2 * th * iters / 4 * 128 / ms / 1e9);
    return 0;
}
