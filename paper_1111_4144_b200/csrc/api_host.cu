// api_host.cu -- host-buffer entry point (include/hpdinv.h: hpdinv_inv_host): a chunked,
// double-buffered H2D -> kernel -> D2H pipeline over caller-owned device workspace.
// Only the upper triangle is transferred host->device for the interleaved layout (the
// kernels never read the strict lower triangle, reading R5), and the result comes back
// in the caller's layout.  Copies run on two internal streams so that H2D of chunk c+1,
// the kernel of chunk c and D2H of chunk c-1 overlap.
//
// Each of the two slots holds: an input region (n*n*chunk elements), an output region of the
// same size and the chunk's info.  Cholesky / LDL run in place on the input region when the
// caller's A and X layout classes agree; otherwise (and always for the non-Hermitian method,
// which is out of place) the kernel writes X in the CALLER'S X layout into the output region,
// so every D2H is one 2-D copy (the kernels accept independent A and X layouts).
// The two copy streams and their events are created once per device and reused by every
// call (serialised by a mutex while a call enqueues its work).
#include <algorithm>
#include <cstdint>
#include <mutex>

#include "../../include/hpdinv.h"

namespace {

struct Slot {
    char* in;        // n*n*chunk elements: A (SoA with ld = chunk, or AoS)
    char* out;       // n*n*chunk elements: X when the kernel runs out of place
    int32_t* info;   // chunk
};

inline int64_t al256(int64_t b) { return (b + 255) / 256 * 256; }

inline int64_t slot_bytes(int n, size_t elem, int64_t chunk) {
    return 2 * al256(int64_t(n) * n * chunk * int64_t(elem)) + al256(chunk * 4);
}

// Per-device copy streams and events, created on first use and kept for the process.
struct Pipe {
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t start = nullptr, in[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr},
                out[2] = {nullptr, nullptr};
    bool ok = false;
};
constexpr int kMaxDev = 64;
std::mutex g_pipe_mu;
Pipe g_pipe[kMaxDev];

// Called with g_pipe_mu held.
cudaError_t get_pipe(Pipe** p) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
    Pipe& q = g_pipe[dev];
    if (!q.ok) {
        auto chk = [&](cudaError_t x) { if (e == cudaSuccess && x != cudaSuccess) e = x; };
        chk(cudaStreamCreateWithFlags(&q.h2d, cudaStreamNonBlocking));
        chk(cudaStreamCreateWithFlags(&q.d2h, cudaStreamNonBlocking));
        chk(cudaEventCreateWithFlags(&q.start, cudaEventDisableTiming));
        for (int s = 0; s < 2; s++) {
            chk(cudaEventCreateWithFlags(&q.in[s], cudaEventDisableTiming));
            chk(cudaEventCreateWithFlags(&q.done[s], cudaEventDisableTiming));
            chk(cudaEventCreateWithFlags(&q.out[s], cudaEventDisableTiming));
        }
        if (e != cudaSuccess) return e;
        q.ok = true;
    }
    *p = &q;
    return cudaSuccess;
}

// method 0 Cholesky, 1 LDL, 2 non-Hermitian; A (strides sm, se) -> X (strides xm, xe), which
// may be A itself (in place) for methods 0 and 1
int launch_inv(int method, int dtype, int64_t m, int n, void* a, int64_t sm, int64_t se,
               void* x, int64_t xm, int64_t xe, int32_t* info, cudaStream_t s) {
    if (dtype == 0) {
        auto* p = static_cast<cuFloatComplex*>(a);
        auto* q = static_cast<cuFloatComplex*>(x);
        if (method == 2) return nonherm_inv_batched_c64(m, n, p, sm, se, q, xm, xe, info, s);
        return method ? ldl_inv_batched_c64(m, n, p, sm, se, q, xm, xe, info, s)
                      : chol_inv_batched_c64(m, n, p, sm, se, q, xm, xe, info, s);
    }
    auto* p = static_cast<cuDoubleComplex*>(a);
    auto* q = static_cast<cuDoubleComplex*>(x);
    if (method == 2) return nonherm_inv_batched_c128(m, n, p, sm, se, q, xm, xe, info, s);
    return method ? ldl_inv_batched_c128(m, n, p, sm, se, q, xm, xe, info, s)
                  : chol_inv_batched_c128(m, n, p, sm, se, q, xm, xe, info, s);
}

int launch_solve_c(int method, int dtype, int64_t m, int n, const void* A, int64_t sAm, int64_t sAe,
                   const void* Y, int64_t sYm, int64_t sYe, void* Xv, int64_t sXm, int64_t sXe,
                   int32_t* info, cudaStream_t s) {
    if (dtype == 0) {
        auto* a = static_cast<const cuFloatComplex*>(A);
        auto* y = static_cast<const cuFloatComplex*>(Y);
        auto* x = static_cast<cuFloatComplex*>(Xv);
        return method ? ldl_solve_batched_c64(m, n, a, sAm, sAe, y, sYm, sYe, x, sXm, sXe, info, s)
                      : chol_solve_batched_c64(m, n, a, sAm, sAe, y, sYm, sYe, x, sXm, sXe, info, s);
    }
    auto* a = static_cast<const cuDoubleComplex*>(A);
    auto* y = static_cast<const cuDoubleComplex*>(Y);
    auto* x = static_cast<cuDoubleComplex*>(Xv);
    return method ? ldl_solve_batched_c128(m, n, a, sAm, sAe, y, sYm, sYe, x, sXm, sXe, info, s)
                  : chol_solve_batched_c128(m, n, a, sAm, sAe, y, sYm, sYe, x, sXm, sXe, info, s);
}

// solve slot: A (n*n*chunk) | y (n*chunk) | x (n*chunk) | info (chunk)
inline int64_t solve_slot_bytes(int n, size_t elem, int64_t chunk) {
    return al256(int64_t(n) * n * chunk * int64_t(elem)) + 2 * al256(int64_t(n) * chunk * int64_t(elem)) + al256(chunk * 4);
}

}  // namespace

extern "C" {

size_t hpdinv_solve_host_workspace_bytes(int dtype, int n, int64_t chunk) {
    if (n < 1 || n > HPDINV_MAX_N || chunk < 1 || dtype < 0 || dtype > 1) return 0;
    return size_t(2 * solve_slot_bytes(n, dtype ? 16 : 8, chunk));
}

int hpdinv_solve_host(int method, int dtype, int64_t batch, int n,
                      const void* A_host, int64_t sAm, int64_t sAe,
                      const void* Y_host, int64_t sYm, int64_t sYe,
                      void* X_host, int64_t sXm, int64_t sXe, int32_t* info_host,
                      void* d_work, size_t work_bytes, int64_t chunk, cudaStream_t stream) {
    if (method < 0 || method > 1) return -1;
    if (dtype < 0 || dtype > 1) return -2;
    if (batch < 0) return -3;
    if (n < 1 || n > HPDINV_MAX_N) return -4;
    if (batch == 0) return 0;
    const size_t elem = dtype ? 16 : 8;
    // n = 1: the element stride addresses nothing (one element per matrix / vector); give it
    // a value that makes the single plane a valid 2-D copy (pitch >= width)
    if (n == 1) { sAe = std::max<int64_t>(sAe, batch); sYe = std::max<int64_t>(sYe, batch); sXe = std::max<int64_t>(sXe, batch); }
    const bool a_soa = sAm == 1 && sAe >= batch;
    const bool a_aos = !a_soa && sAe == 1 && sAm >= int64_t(n) * n;
    const bool y_soa = sYm == 1 && sYe >= batch;
    const bool y_aos = !y_soa && sYe == 1 && sYm >= n;
    const bool x_soa = sXm == 1 && sXe >= batch;
    const bool x_aos = !x_soa && sXe == 1 && sXm >= n;
    if (!A_host) return -5;
    if (!a_soa && !a_aos) return -6;
    if (!Y_host) return -8;
    if (!y_soa && !y_aos) return -9;
    if (!X_host) return -11;
    if (!x_soa && !x_aos) return -12;
    if (!info_host) return -14;
    if (!d_work || reinterpret_cast<uintptr_t>(d_work) % 256) return -15;
    if (chunk <= 0) chunk = std::max<int64_t>(std::min<int64_t>(batch, 4096), (batch + 7) / 8);
    chunk = std::min(chunk, batch);
    while (chunk > 1 && hpdinv_solve_host_workspace_bytes(dtype, n, chunk) > work_bytes) chunk /= 2;
    if (hpdinv_solve_host_workspace_bytes(dtype, n, chunk) > work_bytes) return -16;

    const int64_t sb = solve_slot_bytes(n, elem, chunk);
    const int64_t ab = al256(int64_t(n) * n * chunk * int64_t(elem)), vb = al256(int64_t(n) * chunk * int64_t(elem));
    char* sa[2]; char* sy[2]; char* sx[2]; int32_t* si[2];
    for (int s = 0; s < 2; s++) {
        sa[s] = static_cast<char*>(d_work) + s * sb;
        sy[s] = sa[s] + ab;
        sx[s] = sy[s] + vb;
        si[s] = reinterpret_cast<int32_t*>(sx[s] + vb);
    }
    std::lock_guard<std::mutex> lock(g_pipe_mu);
    Pipe* P = nullptr;
    cudaError_t e = get_pipe(&P);
    if (e != cudaSuccess) return int(e);
    int rc = 0;
    auto chk = [&](cudaError_t x) { if (e == cudaSuccess && x != cudaSuccess) e = x; };
    chk(cudaEventRecord(P->start, stream));
    chk(cudaStreamWaitEvent(P->h2d, P->start, 0));
    chk(cudaStreamWaitEvent(P->d2h, P->start, 0));
    // a previous call (possibly from another user stream, possibly on the same workspace)
    // must have drained its slots before this call refills them
    chk(cudaStreamWaitEvent(P->h2d, P->out[0], 0));
    chk(cudaStreamWaitEvent(P->h2d, P->out[1], 0));
    const char* A = static_cast<const char*>(A_host);
    const char* Y = static_cast<const char*>(Y_host);
    char* X = static_cast<char*>(X_host);
    const int64_t nchunks = (batch + chunk - 1) / chunk;
    for (int64_t c = 0; c < nchunks && e == cudaSuccess && rc == 0; c++) {
        const int s = int(c & 1);
        const int64_t b0 = c * chunk;
        const int64_t m = std::min(chunk, batch - b0);
        if (c >= 2) chk(cudaStreamWaitEvent(P->h2d, P->out[s], 0));
        if (a_soa) {                          // upper planes only, device ld = chunk
            for (int i = 0; i < n; i++)
                chk(cudaMemcpy2DAsync(sa[s] + int64_t(i * n + i) * chunk * elem, chunk * elem,
                                      A + (b0 + int64_t(i * n + i) * sAe) * elem, sAe * elem, m * elem, n - i,
                                      cudaMemcpyHostToDevice, P->h2d));
        } else {
            chk(cudaMemcpy2DAsync(sa[s], int64_t(n) * n * elem, A + b0 * sAm * elem, sAm * elem,
                                  int64_t(n) * n * elem, m, cudaMemcpyHostToDevice, P->h2d));
        }
        if (y_soa)
            chk(cudaMemcpy2DAsync(sy[s], chunk * elem, Y + b0 * elem, sYe * elem, m * elem, n,
                                  cudaMemcpyHostToDevice, P->h2d));
        else
            chk(cudaMemcpy2DAsync(sy[s], int64_t(n) * elem, Y + b0 * sYm * elem, sYm * elem, int64_t(n) * elem, m,
                                  cudaMemcpyHostToDevice, P->h2d));
        chk(cudaEventRecord(P->in[s], P->h2d));
        chk(cudaStreamWaitEvent(stream, P->in[s], 0));
        if (e == cudaSuccess) {
            rc = launch_solve_c(method, dtype, m, n, sa[s], a_soa ? 1 : int64_t(n) * n, a_soa ? chunk : 1,
                                sy[s], y_soa ? 1 : n, y_soa ? chunk : 1, sx[s], x_soa ? 1 : n, x_soa ? chunk : 1,
                                si[s], stream);
        }
        chk(cudaEventRecord(P->done[s], stream));
        chk(cudaStreamWaitEvent(P->d2h, P->done[s], 0));
        if (x_soa)
            chk(cudaMemcpy2DAsync(X + b0 * elem, sXe * elem, sx[s], chunk * elem, m * elem, n,
                                  cudaMemcpyDeviceToHost, P->d2h));
        else
            chk(cudaMemcpy2DAsync(X + b0 * sXm * elem, sXm * elem, sx[s], int64_t(n) * elem, int64_t(n) * elem, m,
                                  cudaMemcpyDeviceToHost, P->d2h));
        chk(cudaMemcpyAsync(info_host + b0, si[s], m * 4, cudaMemcpyDeviceToHost, P->d2h));
        chk(cudaEventRecord(P->out[s], P->d2h));
    }
    const int64_t last = (nchunks - 1) & 1;
    chk(cudaStreamWaitEvent(stream, P->out[last], 0));
    if (nchunks > 1) chk(cudaStreamWaitEvent(stream, P->out[last ^ 1], 0));
    if (rc != 0) return rc;
    return int(e);
}


size_t hpdinv_host_workspace_bytes(int dtype, int n, int64_t chunk) {
    if (n < 1 || n > HPDINV_MAX_N || chunk < 1 || dtype < 0 || dtype > 1) return 0;
    return size_t(2 * slot_bytes(n, dtype ? 16 : 8, chunk));
}

int hpdinv_inv_host(int method, int dtype, int64_t batch, int n,
                    const void* A_host, int64_t sAm, int64_t sAe,
                    void* X_host, int64_t sXm, int64_t sXe, int32_t* info_host,
                    void* d_work, size_t work_bytes, int64_t chunk, cudaStream_t stream) {
    if (method < 0 || method > 2) return -1;
    if (dtype < 0 || dtype > 1) return -2;
    if (batch < 0) return -3;
    if (n < 1 || n > HPDINV_MAX_N) return -4;
    if (batch == 0) return 0;
    const size_t elem = dtype ? 16 : 8;
    // n = 1: the element stride addresses nothing; make the single plane a valid 2-D copy
    if (n == 1) { sAe = std::max<int64_t>(sAe, batch); sXe = std::max<int64_t>(sXe, batch); }
    const bool a_soa = sAm == 1 && sAe >= batch;
    const bool a_aos = !a_soa && sAe == 1 && sAm >= int64_t(n) * n;
    const bool x_soa = sXm == 1 && sXe >= batch;
    const bool x_aos = !x_soa && sXe == 1 && sXm >= int64_t(n) * n;
    if (!A_host) return -5;
    if (!a_soa && !a_aos) return -6;
    if (!X_host) return -8;
    if (!x_soa && !x_aos) return -9;
    if (!info_host) return -11;
    if (!d_work || reinterpret_cast<uintptr_t>(d_work) % 256) return -12;
    if (chunk <= 0) chunk = std::max<int64_t>(std::min<int64_t>(batch, 4096), (batch + 7) / 8);
    chunk = std::min(chunk, batch);
    while (chunk > 1 && hpdinv_host_workspace_bytes(dtype, n, chunk) > work_bytes) chunk /= 2;
    if (hpdinv_host_workspace_bytes(dtype, n, chunk) > work_bytes) return -13;

    const int64_t sb = slot_bytes(n, elem, chunk);
    const int64_t half = al256(int64_t(n) * n * chunk * int64_t(elem));
    Slot slot[2];
    for (int s = 0; s < 2; s++) {
        slot[s].in = static_cast<char*>(d_work) + s * sb;
        slot[s].out = slot[s].in + half;
        slot[s].info = reinterpret_cast<int32_t*>(slot[s].out + half);
    }
    // in place when the layout classes agree (Cholesky / LDL), else out of place into the
    // output region in the caller's X layout; non-Hermitian is always out of place
    const bool inplace = method != 2 && a_soa == x_soa;
    const int64_t dam = a_soa ? 1 : int64_t(n) * n, dae = a_soa ? chunk : 1;
    const int64_t dxm = x_soa ? 1 : int64_t(n) * n, dxe = x_soa ? chunk : 1;

    std::lock_guard<std::mutex> lock(g_pipe_mu);
    Pipe* P = nullptr;
    cudaError_t e = get_pipe(&P);
    if (e != cudaSuccess) return int(e);
    int rc = 0;
    auto chk = [&](cudaError_t x) { if (e == cudaSuccess && x != cudaSuccess) e = x; };
    // everything starts after prior work on `stream`
    chk(cudaEventRecord(P->start, stream));
    chk(cudaStreamWaitEvent(P->h2d, P->start, 0));
    chk(cudaStreamWaitEvent(P->d2h, P->start, 0));
    // a previous call (possibly from another user stream, possibly on the same workspace)
    // must have drained its slots before this call refills them
    chk(cudaStreamWaitEvent(P->h2d, P->out[0], 0));
    chk(cudaStreamWaitEvent(P->h2d, P->out[1], 0));

    const char* A = static_cast<const char*>(A_host);
    char* X = static_cast<char*>(X_host);
    const int64_t nchunks = (batch + chunk - 1) / chunk;
    for (int64_t c = 0; c < nchunks && e == cudaSuccess && rc == 0; c++) {
        const int s = int(c & 1);
        const int64_t b0 = c * chunk;
        const int64_t m = std::min(chunk, batch - b0);
        if (c >= 2) chk(cudaStreamWaitEvent(P->h2d, P->out[s], 0));   // slot s drained
        // ---- H2D: the device input is interleaved (ld = chunk) when the host A is, else AoS
        char* res = inplace ? slot[s].in : slot[s].out;
        if (a_soa && method == 2) {         // non-Hermitian: every plane of D
            chk(cudaMemcpy2DAsync(slot[s].in, chunk * elem, A + b0 * elem, sAe * elem, m * elem, int64_t(n) * n,
                                  cudaMemcpyHostToDevice, P->h2d));
        } else if (a_soa) {
            for (int i = 0; i < n; i++) {   // planes (i, i..n-1): only the upper triangle
                const char* src = A + (b0 + int64_t(i * n + i) * sAe) * elem;
                char* dst = slot[s].in + int64_t(i * n + i) * chunk * elem;
                chk(cudaMemcpy2DAsync(dst, chunk * elem, src, sAe * elem, m * elem, n - i,
                                      cudaMemcpyHostToDevice, P->h2d));
            }
        } else {
            chk(cudaMemcpy2DAsync(slot[s].in, int64_t(n) * n * elem, A + b0 * sAm * elem, sAm * elem,
                                  int64_t(n) * n * elem, m, cudaMemcpyHostToDevice, P->h2d));
        }
        chk(cudaEventRecord(P->in[s], P->h2d));
        // ---- kernel
        chk(cudaStreamWaitEvent(stream, P->in[s], 0));
        if (e == cudaSuccess)
            rc = launch_inv(method, dtype, m, n, slot[s].in, dam, dae, res, inplace ? dam : dxm,
                            inplace ? dae : dxe, slot[s].info, stream);
        chk(cudaEventRecord(P->done[s], stream));
        // ---- D2H: the device result is already in the caller's layout class, one 2-D copy
        chk(cudaStreamWaitEvent(P->d2h, P->done[s], 0));
        if (x_soa)
            chk(cudaMemcpy2DAsync(X + b0 * elem, sXe * elem, res, chunk * elem, m * elem,
                                  int64_t(n) * n, cudaMemcpyDeviceToHost, P->d2h));
        else
            chk(cudaMemcpy2DAsync(X + b0 * sXm * elem, sXm * elem, res, int64_t(n) * n * elem,
                                  int64_t(n) * n * elem, m, cudaMemcpyDeviceToHost, P->d2h));
        chk(cudaMemcpyAsync(info_host + b0, slot[s].info, m * 4, cudaMemcpyDeviceToHost, P->d2h));
        chk(cudaEventRecord(P->out[s], P->d2h));
    }
    // the caller's stream observes completion of the whole pipeline
    const int64_t last = (nchunks - 1) & 1;
    chk(cudaStreamWaitEvent(stream, P->out[last], 0));
    if (nchunks > 1) chk(cudaStreamWaitEvent(stream, P->out[last ^ 1], 0));
    if (rc != 0) return rc;
    return int(e);
}

}  // extern "C"
