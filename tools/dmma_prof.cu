// dmma_prof.cu -- per-phase cycle breakdown of k_dmma (lane 0 of every warp, clock64 marks),
// built with -DHPDINV_DMMA_PROF.  Input: one well-conditioned HPD matrix replicated over the
// batch -- timing only, numerics are not checked here.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHPDINV_DMMA_PROF tools/dmma_prof.cu -o tools/dmma_prof
#include <cstdio>
#include <vector>
#include "../paper_1111_4144_b200/csrc/k_dmma.cuh"
using namespace hpdinv;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const int64_t batch = argc > 1 ? atoll(argv[1]) : (1 << 16);
    const int N = 64;
    std::vector<double2> h(size_t(N) * N);
    for (int i = 0; i < N; i++)
        for (int j = 0; j < N; j++) {
            double2 v;
            v.x = (i == j) ? 2.0 * N : double(((i * 7 + j * 3) % 11) - 5) / 11.0;
            v.y = (i == j) ? 0.0 : double(((i * 5 + j * 13) % 7) - 3) / 7.0 * (i < j ? 1 : -1);
            h[size_t(i) * N + j] = v;
        }
    double2 *A, *X;
    int* info;
    cudaMalloc(&A, sizeof(double2) * N * N * batch);
    cudaMalloc(&X, sizeof(double2) * N * N * batch);
    cudaMalloc(&info, 4 * batch);
    for (int64_t b = 0; b < batch; b++) cudaMemcpy(A + b * N * N, h.data(), sizeof(double2) * N * N, cudaMemcpyHostToDevice);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeTiledFn enc = reinterpret_cast<EncodeTiledFn>(p);
    CUtensorMap tm;
    const cuuint64_t dims[3] = {128, 64, cuuint64_t(batch)};
    const cuuint64_t strides[2] = {64 * 16, 64 * 64 * 16};
    const cuuint32_t box[3] = {16, 8, 1}, es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap tx;                                   // X by TMA bulk stores, as the library does
    enc(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int grid = int(batch < 148 * 6 ? (batch + 5) / 6 : 148);
    cudaFuncSetAttribute(k_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, dm::SMEM);
    k_dmma<<<grid, dm::NT, dm::SMEM>>>(tm, tx, 1, batch, X, N * N, 1, info);
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(dm::g_prof, z, sizeof(unsigned long long) * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_dmma<<<grid, dm::NT, dm::SMEM>>>(tm, tx, 1, batch, X, N * N, 1, info);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long pr2[2][16] = {};
    cudaMemcpyFromSymbol(pr2[0], dm::g_prof, sizeof(unsigned long long) * 16);
    const char* names[2][10] = {{"wait", "F1diag", "F2a", "F1+F2b", "I1", "I2+I3", "I4", "S5", "other", "-"}, {"", "", "", "", "", "", "", "", "", ""}};
    printf("k_dmma batch=%lld %.3f ms (%s): %.0f cycles per matrix per SM\n", (long long)batch, ms,
           cudaGetErrorString(cudaGetLastError()), ms * 1e-3 * 1.965e9 * 148 / batch);
    for (int role = 0; role < 2; role++) {
        unsigned long long tot = 0;
        for (int i = 0; i < 10; i++) tot += pr2[role][i];
        printf(" %s warp: %.0f cycles per matrix\n", role ? "GEMM" : "serial", double(tot) / batch);
        for (int i = 0; i < 10; i++)
            if (pr2[role][i]) printf("  %-16s %9.0f cyc/matrix  %5.1f %%\n", names[role][i], double(pr2[role][i]) / batch, 100.0 * pr2[role][i] / tot);
    }
    return 0;
}
