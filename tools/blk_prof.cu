// blk_prof.cu -- per-phase cycle breakdown of k_blk (thread 0 of every CTA, clock64 marks),
// built with -DHPDINV_BLK_PROF.  Inputs: one well-conditioned HPD matrix (diagonally dominant,
// deterministic) replicated over the batch -- timing only, no numerics are checked here.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHPDINV_BLK_PROF tools/blk_prof.cu -o tools/blk_prof
#include <cstdio>
#include <vector>
#include "../paper_1111_4144_b200/csrc/k_blk.cuh"
using namespace hpdinv;

template <typename T, int N, int NB, bool LDL, int NT, int RT>
void run(const char* name, int64_t batch) {
    using V = cplx<T>;
    using Sh = BlkShape<T, N, NB, NT, RT>;
    std::vector<V> h(size_t(N) * N);
    for (int i = 0; i < N; i++)
        for (int j = 0; j < N; j++) {
            V v; v.x = (i == j) ? T(2 * N) : T(((i * 7 + j * 3) % 11) - 5) / T(11);
            v.y = (i == j) ? T(0) : T(((i * 5 + j * 13) % 7) - 3) / T(7) * (i < j ? 1 : -1);
            h[size_t(i) * N + j] = v;
        }
    V *A, *X; int* info;
    cudaMalloc(&A, sizeof(V) * N * N * batch);
    cudaMalloc(&X, sizeof(V) * N * N * batch);
    cudaMalloc(&info, 4 * batch);
    for (int64_t b = 0; b < batch; b++) cudaMemcpy(A + b * N * N, h.data(), sizeof(V) * N * N, cudaMemcpyHostToDevice);
    auto fn = k_blk<T, N, NB, LDL, NT, RT>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Sh::smem_bytes));
    fn<<<unsigned(batch), NT, Sh::smem_bytes>>>(batch, A, N * N, 1, X, N * N, 1, info);   // warm-up
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(blk::g_prof, z, sizeof(z));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fn<<<unsigned(batch), NT, Sh::smem_bytes>>>(batch, A, N * N, 1, X, N * N, 1, info);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long p[32];
    cudaMemcpyFromSymbol(p, blk::g_prof, sizeof(p));
    const char* names[10] = {"F1", "F2a", "F2b", "I1", "I2", "I3", "I4", "S5", "-", "S1"};
    for (int role = 0; role < (NT > 32 ? 2 : 1); role++) {
        unsigned long long tot = 0;
        for (int i = 0; i < 10; i++) tot += p[role * 16 + i];
        printf("%s batch=%lld  %.3f ms  (%s)  %s warp, cycles/matrix (lane 0): %.0f\n", name, (long long)batch, ms,
               cudaGetErrorString(cudaGetLastError()), role == 0 ? "serial" : "GEMM", double(tot) / batch);
        for (int i = 0; i < 10; i++)
            if (p[role * 16 + i])
                printf("  %-4s %9.0f cyc/matrix  %5.1f %%\n", names[i], double(p[role * 16 + i]) / batch,
                       100.0 * p[role * 16 + i] / tot);
    }
    cudaFree(A); cudaFree(X); cudaFree(info);
}

int main() {
    run<double, 64, 8, false, 128, 2>("c128 n=64 chol NB=8 NT=128", 1 << 16);
    run<float, 32, 8, true, 32, 2>("c64 n=32 ldl NB=8 NT=32", 1 << 18);
    return 0;
}
