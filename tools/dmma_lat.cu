// dmma_lat.cu -- latency / per-warp throughput of DMMA (m8n8k4 f64), DFMA and SHFL on sm_100a,
// to size the ILP the one-matrix-per-warp kernel (k_dmma) needs.
//   chain<A>: A independent accumulators, each a dependent DMMA chain, ONE warp per SM
//             sub-partition (4 warps per SM) -> cycles per DMMA issue at that ILP
//   warps<W>: W warps per SM, 8 independent accumulators each -> saturation
//   dfma_chain / shfl_chain: dependent latency
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int A>
__global__ void chain(double* out, long long* cyc, int iters) {
    double c[A][2];
    for (int k = 0; k < A; k++) { c[k][0] = threadIdx.x; c[k][1] = 1; }
    const double a = 1e-3 * threadIdx.x, b = 0.5;
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < A; k++) dmma(c[k][0], c[k][1], a, b);
    long long t1 = clock64();
    double s = 0;
    for (int k = 0; k < A; k++) s += c[k][0] + c[k][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void dfma_chain(double* out, long long* cyc, int iters) {
    double x = threadIdx.x;
    const double a = 0.999, b = 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 16; u++) x = fma(x, a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void shfl_chain(double* out, long long* cyc, int iters) {
    int v = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 16; u++) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
    }
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lds_chain(double* out, long long* cyc, int iters) {
    __shared__ int buf[64];
    buf[threadIdx.x] = (threadIdx.x + 1) & 31;
    __syncwarp();
    int v = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 16; u++) v = buf[v];
    }
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <typename F>
double run(F f) {
    long long* cyc;
    cudaMalloc(&cyc, 8);
    f(cyc);
    cudaDeviceSynchronize();
    f(cyc);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    cudaFree(cyc);
    return double(h);
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 24);
    const int it = 1024;
    printf("{");
    // one warp per SMSP: 148 CTAs x 4 warps (one CTA per SM via large smem is not needed: 4 warps/CTA)
#define CH(A)                                                                                    \
    {                                                                                            \
        double c = run([&](long long* cy) { chain<A><<<148, 128>>>(out, cy, it); });             \
        printf("\"dmma_cyc_per_issue_1warp_ilp%d\": %.2f, ", A, c / (it * double(A)));           \
    }
    CH(1) CH(2) CH(4) CH(8) CH(16)
#undef CH
    {
        double c = run([&](long long* cy) { chain<8><<<148, 64>>>(out, cy, it); });
        printf("\"dmma_cyc_per_issue_halfwarp_per_smsp_ilp8\": %.2f, ", c / (it * 8.0));
        c = run([&](long long* cy) { chain<8><<<148, 256>>>(out, cy, it); });
        printf("\"dmma_cyc_per_issue_2warps_per_smsp_ilp8\": %.2f, ", c / (it * 8.0));
    }
    double c = run([&](long long* cy) { dfma_chain<<<1, 32>>>(out, cy, it); });
    printf("\"dfma_latency\": %.2f, ", c / (it * 16.0));
    c = run([&](long long* cy) { shfl_chain<<<1, 32>>>(out, cy, it); });
    printf("\"shfl_latency\": %.2f, ", c / (it * 16.0));
    c = run([&](long long* cy) { lds_chain<<<1, 32>>>(out, cy, it); });
    printf("\"lds_latency\": %.2f}\n", c / (it * 16.0));
    return 0;
}
