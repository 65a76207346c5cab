// api_host.cu -- host-buffer entry point (include/hpdinv.h: hpdinv_inv_host): a chunked,
// double-buffered H2D -> kernel -> D2H pipeline over caller-owned device workspace.
// Only the upper triangle is transferred host->device for the interleaved layout (the
// kernels never read the strict lower triangle, reading R5), and the result comes back
// in the caller's layout.  Copies run on two internal streams so that H2D of chunk c+1,
// the kernel of chunk c and D2H of chunk c-1 overlap.
#include <algorithm>
#include <cstdint>

#include "../../include/hpdinv.h"

namespace {

struct Slot {
    char* buf;       // n*n*chunk elements (A in, X out: the kernel runs in place)
    int32_t* info;   // chunk
};

inline int64_t slot_bytes(int n, size_t elem, int64_t chunk) {
    int64_t b = int64_t(n) * n * chunk * int64_t(elem);
    b = (b + 255) / 256 * 256;
    return b + (chunk * 4 + 255) / 256 * 256;
}

// method 0 Cholesky, 1 LDL (in place), 2 non-Hermitian (out of place into `out`)
int launch_inv(int method, int dtype, int64_t m, int n, void* buf, int64_t sm, int64_t se,
               int32_t* info, cudaStream_t s, void* out = nullptr) {
    if (dtype == 0) {
        auto* p = static_cast<cuFloatComplex*>(buf);
        if (method == 2) return nonherm_inv_batched_c64(m, n, p, sm, se, static_cast<cuFloatComplex*>(out), sm, se, info, s);
        return method ? ldl_inv_batched_c64(m, n, p, sm, se, p, sm, se, info, s)
                      : chol_inv_batched_c64(m, n, p, sm, se, p, sm, se, info, s);
    }
    auto* p = static_cast<cuDoubleComplex*>(buf);
    if (method == 2) return nonherm_inv_batched_c128(m, n, p, sm, se, static_cast<cuDoubleComplex*>(out), sm, se, info, s);
    return method ? ldl_inv_batched_c128(m, n, p, sm, se, p, sm, se, info, s)
                  : chol_inv_batched_c128(m, n, p, sm, se, p, sm, se, info, s);
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

inline int64_t al256(int64_t b) { return (b + 255) / 256 * 256; }

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
    const bool a_soa = (sAm == 1 && sAe >= batch) || (n == 1 && sAm == 1);
    const bool a_aos = !a_soa && sAe == 1 && sAm >= int64_t(n) * n;
    const bool y_soa = (sYm == 1 && sYe >= batch) || (n == 1 && sYm == 1);
    const bool y_aos = !y_soa && sYe == 1 && sYm >= n;
    const bool x_soa = (sXm == 1 && sXe >= batch) || (n == 1 && sXm == 1);
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
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_start = nullptr, ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr},
                ev_out[2] = {nullptr, nullptr};
    cudaError_t e = cudaSuccess;
    int rc = 0;
    auto chk = [&](cudaError_t x) { if (e == cudaSuccess && x != cudaSuccess) e = x; };
    chk(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    chk(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    chk(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
    for (int s = 0; s < 2; s++) {
        chk(cudaEventCreateWithFlags(&ev_in[s], cudaEventDisableTiming));
        chk(cudaEventCreateWithFlags(&ev_done[s], cudaEventDisableTiming));
        chk(cudaEventCreateWithFlags(&ev_out[s], cudaEventDisableTiming));
    }
    chk(cudaEventRecord(ev_start, stream));
    chk(cudaStreamWaitEvent(h2d, ev_start, 0));
    chk(cudaStreamWaitEvent(d2h, ev_start, 0));
    const char* A = static_cast<const char*>(A_host);
    const char* Y = static_cast<const char*>(Y_host);
    char* X = static_cast<char*>(X_host);
    const int64_t nchunks = (batch + chunk - 1) / chunk;
    for (int64_t c = 0; c < nchunks && e == cudaSuccess && rc == 0; c++) {
        const int s = int(c & 1);
        const int64_t b0 = c * chunk;
        const int64_t m = std::min(chunk, batch - b0);
        if (c >= 2) chk(cudaStreamWaitEvent(h2d, ev_out[s], 0));
        if (a_soa) {                          // upper planes only, device ld = chunk
            for (int i = 0; i < n; i++)
                chk(cudaMemcpy2DAsync(sa[s] + int64_t(i * n + i) * chunk * elem, chunk * elem,
                                      A + (b0 + int64_t(i * n + i) * sAe) * elem, sAe * elem, m * elem, n - i,
                                      cudaMemcpyHostToDevice, h2d));
        } else {
            chk(cudaMemcpy2DAsync(sa[s], int64_t(n) * n * elem, A + b0 * sAm * elem, sAm * elem,
                                  int64_t(n) * n * elem, m, cudaMemcpyHostToDevice, h2d));
        }
        if (y_soa)
            chk(cudaMemcpy2DAsync(sy[s], chunk * elem, Y + b0 * elem, sYe * elem, m * elem, n,
                                  cudaMemcpyHostToDevice, h2d));
        else
            chk(cudaMemcpy2DAsync(sy[s], int64_t(n) * elem, Y + b0 * sYm * elem, sYm * elem, int64_t(n) * elem, m,
                                  cudaMemcpyHostToDevice, h2d));
        chk(cudaEventRecord(ev_in[s], h2d));
        chk(cudaStreamWaitEvent(stream, ev_in[s], 0));
        if (e == cudaSuccess) {
            rc = launch_solve_c(method, dtype, m, n, sa[s], a_soa ? 1 : int64_t(n) * n, a_soa ? chunk : 1,
                                sy[s], y_soa ? 1 : n, y_soa ? chunk : 1, sx[s], x_soa ? 1 : n, x_soa ? chunk : 1,
                                si[s], stream);
        }
        chk(cudaEventRecord(ev_done[s], stream));
        chk(cudaStreamWaitEvent(d2h, ev_done[s], 0));
        if (x_soa)
            chk(cudaMemcpy2DAsync(X + b0 * elem, sXe * elem, sx[s], chunk * elem, m * elem, n,
                                  cudaMemcpyDeviceToHost, d2h));
        else
            chk(cudaMemcpy2DAsync(X + b0 * sXm * elem, sXm * elem, sx[s], int64_t(n) * elem, int64_t(n) * elem, m,
                                  cudaMemcpyDeviceToHost, d2h));
        chk(cudaMemcpyAsync(info_host + b0, si[s], m * 4, cudaMemcpyDeviceToHost, d2h));
        chk(cudaEventRecord(ev_out[s], d2h));
    }
    const int64_t last = (nchunks - 1) & 1;
    chk(cudaStreamWaitEvent(stream, ev_out[last], 0));
    if (nchunks > 1) chk(cudaStreamWaitEvent(stream, ev_out[last ^ 1], 0));
    for (int s = 0; s < 2; s++) {
        if (ev_in[s]) cudaEventDestroy(ev_in[s]);
        if (ev_done[s]) cudaEventDestroy(ev_done[s]);
        if (ev_out[s]) cudaEventDestroy(ev_out[s]);
    }
    if (ev_start) cudaEventDestroy(ev_start);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
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
    const bool a_soa = (sAm == 1 && sAe >= batch) || (n == 1 && sAm == 1);
    const bool a_aos = !a_soa && sAe == 1 && sAm >= int64_t(n) * n;
    const bool x_soa = (sXm == 1 && sXe >= batch) || (n == 1 && sXm == 1);
    const bool x_aos = !x_soa && sXe == 1 && sXm >= int64_t(n) * n;
    if (!A_host) return -5;
    if (!a_soa && !a_aos) return -6;
    if (!X_host) return -8;
    if (!x_soa && !x_aos) return -9;
    if (!info_host) return -11;
    if (!d_work) return -12;
    if (chunk <= 0) chunk = std::max<int64_t>(std::min<int64_t>(batch, 4096), (batch + 7) / 8);
    chunk = std::min(chunk, batch);
    while (chunk > 1 && hpdinv_host_workspace_bytes(dtype, n, chunk) > work_bytes) chunk /= 2;
    if (hpdinv_host_workspace_bytes(dtype, n, chunk) > work_bytes) return -13;
    if (reinterpret_cast<uintptr_t>(d_work) % 256) return -12;

    const int64_t sb = slot_bytes(n, elem, chunk);
    // method 2 (non-Hermitian) is out of place: half a slot in, half out, chunk / 2 per step
    const bool nh = method == 2;
    const int64_t cbuf = chunk;
    if (nh) chunk = std::max<int64_t>(1, chunk / 2);
    Slot slot[2];
    for (int s = 0; s < 2; s++) {
        slot[s].buf = static_cast<char*>(d_work) + s * sb;
        slot[s].info = reinterpret_cast<int32_t*>(slot[s].buf + (int64_t(n) * n * cbuf * int64_t(elem) + 255) / 256 * 256);
    }

    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_start = nullptr, ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr},
                ev_out[2] = {nullptr, nullptr};
    cudaError_t e = cudaSuccess;
    int rc = 0;
    auto chk = [&](cudaError_t x) { if (e == cudaSuccess && x != cudaSuccess) e = x; };
    chk(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    chk(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    chk(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
    for (int s = 0; s < 2; s++) {
        chk(cudaEventCreateWithFlags(&ev_in[s], cudaEventDisableTiming));
        chk(cudaEventCreateWithFlags(&ev_done[s], cudaEventDisableTiming));
        chk(cudaEventCreateWithFlags(&ev_out[s], cudaEventDisableTiming));
    }
    // everything starts after prior work on `stream`
    chk(cudaEventRecord(ev_start, stream));
    chk(cudaStreamWaitEvent(h2d, ev_start, 0));
    chk(cudaStreamWaitEvent(d2h, ev_start, 0));

    const char* A = static_cast<const char*>(A_host);
    char* X = static_cast<char*>(X_host);
    const int64_t nchunks = (batch + chunk - 1) / chunk;
    for (int64_t c = 0; c < nchunks && e == cudaSuccess && rc == 0; c++) {
        const int s = int(c & 1);
        const int64_t b0 = c * chunk;
        const int64_t m = std::min(chunk, batch - b0);
        if (c >= 2) chk(cudaStreamWaitEvent(h2d, ev_out[s], 0));   // slot s drained
        // ---- H2D: device slot is interleaved (ld = chunk) when the host A is, else AoS
        char* res = nh ? slot[s].buf + int64_t(n) * n * chunk * int64_t(elem) : slot[s].buf;
        if (a_soa && nh) {                  // non-Hermitian: every plane of D
            chk(cudaMemcpy2DAsync(slot[s].buf, chunk * elem, A + b0 * elem, sAe * elem, m * elem, int64_t(n) * n,
                                  cudaMemcpyHostToDevice, h2d));
        } else if (a_soa) {
            for (int i = 0; i < n; i++) {   // planes (i, i..n-1): only the upper triangle
                const char* src = A + (b0 + int64_t(i * n + i) * sAe) * elem;
                char* dst = slot[s].buf + int64_t(i * n + i) * chunk * elem;
                chk(cudaMemcpy2DAsync(dst, chunk * elem, src, sAe * elem, m * elem, n - i,
                                      cudaMemcpyHostToDevice, h2d));
            }
        } else {
            chk(cudaMemcpy2DAsync(slot[s].buf, int64_t(n) * n * elem, A + b0 * sAm * elem, sAm * elem,
                                  int64_t(n) * n * elem, m, cudaMemcpyHostToDevice, h2d));
        }
        chk(cudaEventRecord(ev_in[s], h2d));
        // ---- kernel, in place on the slot
        chk(cudaStreamWaitEvent(stream, ev_in[s], 0));
        if (e == cudaSuccess) {
            rc = a_soa ? launch_inv(method, dtype, m, n, slot[s].buf, 1, chunk, slot[s].info, stream, res)
                       : launch_inv(method, dtype, m, n, slot[s].buf, int64_t(n) * n, 1, slot[s].info, stream, res);
        }
        chk(cudaEventRecord(ev_done[s], stream));
        // ---- D2H into the caller's layout
        chk(cudaStreamWaitEvent(d2h, ev_done[s], 0));
        const int64_t dsm = a_soa ? 1 : int64_t(n) * n, dse = a_soa ? chunk : 1;
        if (x_soa && a_soa) {
            chk(cudaMemcpy2DAsync(X + b0 * elem, sXe * elem, res, chunk * elem, m * elem,
                                  int64_t(n) * n, cudaMemcpyDeviceToHost, d2h));
        } else if (x_aos && !a_soa) {
            chk(cudaMemcpy2DAsync(X + b0 * sXm * elem, sXm * elem, res, int64_t(n) * n * elem,
                                  int64_t(n) * n * elem, m, cudaMemcpyDeviceToHost, d2h));
        } else {
            // mixed layouts: element-plane / matrix scatter with 2-D copies (one per element)
            for (int64_t el = 0; el < int64_t(n) * n; el++)
                chk(cudaMemcpy2DAsync(X + (b0 * sXm + el * sXe) * elem, sXm * elem,
                                      res + el * dse * elem, dsm * elem, elem, m,
                                      cudaMemcpyDeviceToHost, d2h));
        }
        chk(cudaMemcpyAsync(info_host + b0, slot[s].info, m * 4, cudaMemcpyDeviceToHost, d2h));
        chk(cudaEventRecord(ev_out[s], d2h));
    }
    // the caller's stream observes completion of the whole pipeline
    const int64_t last = (nchunks - 1) & 1;
    chk(cudaStreamWaitEvent(stream, ev_out[last], 0));
    if (nchunks > 1) chk(cudaStreamWaitEvent(stream, ev_out[last ^ 1], 0));
    // resources are released once the device is done with them (CUDA semantics)
    for (int s = 0; s < 2; s++) {
        if (ev_in[s]) cudaEventDestroy(ev_in[s]);
        if (ev_done[s]) cudaEventDestroy(ev_done[s]);
        if (ev_out[s]) cudaEventDestroy(ev_out[s]);
    }
    if (ev_start) cudaEventDestroy(ev_start);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
    if (rc != 0) return rc;
    return int(e);
}

}  // extern "C"
