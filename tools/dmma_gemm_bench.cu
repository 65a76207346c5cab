// dmma_gemm_bench.cu -- per-warp DMMA issue rate for the k_dmma GEMM pattern: NT complex 8x8
// accumulator tiles, each k-step one A fragment + NT B fragments loaded from shared memory
// (LDS.128, swizzled slots) and 4 DMMA per tile; one warp per SM sub-partition.
// Prints cycles per DMMA for NT = 1..7 and for the split-halves issue order.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
struct CAcc { double r0, r1, i0, i1; };

template <int NT, bool SPLIT>
__global__ void kern(double* out, long long* cyc, int steps) {
    __shared__ double2 sm[4][64 * 8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = lane; i < 64 * 8; i += 32) sm[warp][i] = make_double2(1e-3 * i, 2e-3 * i);
    __syncwarp();
    const double2* T = sm[warp];
    const int r = lane >> 2, q = lane & 3;
    const int oa = r * 8 + ((2 * q) ^ r), ob = (2 * q) * 8 + (r ^ (2 * q));
    CAcc a[NT];
    for (int u = 0; u < NT; u++) a[u] = CAcc{0, 0, 0, 0};
    long long t0 = clock64();
    for (int st = 0; st < steps; st++) {
        const int base = (st & 7) * 64;
        const double2 w = T[base + oa];
        double2 x[NT];
#pragma unroll
        for (int u = 0; u < NT; u++) x[u] = T[((base + 64 * (u + 1)) & (64 * 8 - 1)) + ob];
        const double nwi = -w.y;
        if (SPLIT) {
#pragma unroll
            for (int u = 0; u < NT; u++) { dmma(a[u].r0, a[u].r1, w.x, x[u].x); dmma(a[u].i0, a[u].i1, w.x, x[u].y); }
#pragma unroll
            for (int u = 0; u < NT; u++) { dmma(a[u].r0, a[u].r1, nwi, x[u].y); dmma(a[u].i0, a[u].i1, w.y, x[u].x); }
        } else {
#pragma unroll
            for (int u = 0; u < NT; u++) {
                dmma(a[u].r0, a[u].r1, w.x, x[u].x); dmma(a[u].i0, a[u].i1, w.x, x[u].y);
                dmma(a[u].r0, a[u].r1, nwi, x[u].y); dmma(a[u].i0, a[u].i1, w.y, x[u].x);
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int u = 0; u < NT; u++) s += a[u].r0 + a[u].r1 + a[u].i0 + a[u].i1;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int NT, bool SPLIT>
void run(double* out, long long* cyc, int warps) {
    const int steps = 4096;
    kern<NT, SPLIT><<<148, 32 * warps>>>(out, cyc, steps);
    kern<NT, SPLIT><<<148, 32 * warps>>>(out, cyc, steps);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("\"nt%d_%s_w%d\": %.2f, ", NT, SPLIT ? "split" : "seq", warps, double(h) / (steps * 4.0 * NT));
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 8);
    printf("{");
    run<1, false>(out, cyc, 4); run<2, false>(out, cyc, 4); run<4, false>(out, cyc, 4); run<7, false>(out, cyc, 4);
    run<1, true>(out, cyc, 4); run<2, true>(out, cyc, 4); run<4, true>(out, cyc, 4); run<7, true>(out, cyc, 4);
    run<7, true>(out, cyc, 2);
    printf("\"done\": 1}\n");
    return 0;
}
