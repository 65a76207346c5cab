/*
 * hpdinv.h -- C ABI of the B200-native batched HPD inversion library (libhpdinv.so).
 *
 * Implements, for many small complex Hermitian positive-definite (HPD) matrices at once,
 * the method of "Matrix Inversion Using Cholesky Decomposition" (arxiv/paper_1111_4144;
 * citations P:<line> = PAPER.md line):
 *
 *   1. in-place Cholesky A = R*R, eqs. (3)-(4), P:37-45            (chol_*)
 *      or the square-root-free LDL A = R*DR, eqs. (10)-(11), P:77-85 (ldl_*);
 *   2. the proposed direct inversion, eqs. (20)-(24), P:151-178 (LDL: eqs. (25)-(29),
 *      P:182-204): the forward solve R*B = I (eq. 22) is skipped because the upper part of
 *      B is S = diag(1/r_ii) (eq. 24; S~ = diag(1/d_i), eq. 29), and only the upper half of
 *      X = A^-1 is back-substituted from R x_i = s_i;
 *   3. the Hermitian mirror x_ji = conj(x_ij).
 *
 * All work runs in hand-written sm_100a CUDA kernels; there is no CPU fallback.
 *
 * ---------------------------------------------------------------------------------------
 * Common conventions (all entry points)
 * ---------------------------------------------------------------------------------------
 * Addressing.  Element (i, j) (0-based, row-major as in P:33) of matrix b (0 <= b < batch)
 *   is at  base[b * stride_mat + (i * n + j) * stride_elem]  (strides in ELEMENTS).
 *   Two layout classes are accepted:
 *     - interleaved / SoA:  stride_mat == 1 and stride_elem >= batch  (element plane e is
 *       contiguous across the batch; the layout of configs 1-3);
 *     - contiguous / AoS:   stride_elem == 1 and stride_mat >= n*n   (each matrix is one
 *       contiguous n*n block; configs 4-5).
 *   For n == 1 any stride_mat >= 1 with stride_elem >= 1 is accepted.  A and X may use
 *   different classes.
 * What is read.  Only the upper triangle a_ij, i <= j (eqs. 3-4 and 10-11 never index
 *   i > j); Im(a_ii) is ignored.  The strict lower triangle is never read and need not be
 *   valid (LAPACK uplo='U' semantics).  No Hermitian validation is done.
 * What is written.  All n*n entries of X_b: x_ji == conj(x_ij) bit-for-bit, Im(x_ii) == +0,
 *   and info[b].  When info[b] != 0, every entry of X_b is NaN.
 * info (int32, device, length batch).  0 = success.  k in [1, n] = first 1-based pivot with
 *   !(t_k > 0), t_k = Re a_kk - sum_{i<k} |r_ik|^2 the radicand of eq. (3) (LDL: !(d_k > 0),
 *   eq. (10)); NaN pivots are flagged.  In exact arithmetic t_k = d_k, so both methods flag
 *   the same k.
 * Aliasing.  X == A with identical strides (in-place, the spirit of P:45) is supported;
 *   any other overlap is undefined.
 * Precision.  c64 computes in fp32, c128 in fp64 (no mixed precision, no tensor cores).
 * Ownership.  The caller owns every buffer.  The library allocates no device memory and
 *   keeps no per-call state; calls are reentrant and thread-safe.
 * Streams.  Work is enqueued on `stream` (0 = legacy default stream) and returns
 *   immediately; results are valid once the stream reaches that point.
 * Supported n.  1 <= n <= 64.
 * Return value.  0 = enqueued (or nothing to do when batch == 0).
 *   -k = argument k (1-based position in the signature) is invalid: batch < 0; n outside
 *   [1, 64]; NULL pointer with batch > 0; unsupported stride combination; pointer not
 *   aligned to its element size.  Nothing is launched in that case.
 *   > 0 = a cudaError_t reported by the kernel launch.
 * No C++ exception crosses this ABI.
 */
#ifndef HPDINV_H
#define HPDINV_H

#include <stddef.h>
#include <stdint.h>

#include <cuComplex.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPDINV_MAX_N 64

/* Cholesky (eqs. 3-4) + proposed inversion (eqs. 20-24) + mirror, complex64 / fp32.
 * Args: 1 batch, 2 n, 3 A, 4 strideA_mat, 5 strideA_elem, 6 X, 7 strideX_mat,
 *       8 strideX_elem, 9 info, 10 stream. */
int chol_inv_batched_c64(int64_t batch, int n,
                         const cuFloatComplex *A, int64_t strideA_mat, int64_t strideA_elem,
                         cuFloatComplex *X, int64_t strideX_mat, int64_t strideX_elem,
                         int32_t *info, cudaStream_t stream);

/* Same, complex128 / fp64. */
int chol_inv_batched_c128(int64_t batch, int n,
                          const cuDoubleComplex *A, int64_t strideA_mat, int64_t strideA_elem,
                          cuDoubleComplex *X, int64_t strideX_mat, int64_t strideX_elem,
                          int32_t *info, cudaStream_t stream);

/* LDL (eqs. 10-11, square-root free) + proposed inversion with unit R and S~ = diag(1/d_i)
 * (eqs. 25-29) + mirror, complex64 / fp32. Same arguments as chol_inv_batched_c64. */
int ldl_inv_batched_c64(int64_t batch, int n,
                        const cuFloatComplex *A, int64_t strideA_mat, int64_t strideA_elem,
                        cuFloatComplex *X, int64_t strideX_mat, int64_t strideX_elem,
                        int32_t *info, cudaStream_t stream);

/* Same, complex128 / fp64. */
int ldl_inv_batched_c128(int64_t batch, int n,
                         const cuDoubleComplex *A, int64_t strideA_mat, int64_t strideA_elem,
                         cuDoubleComplex *X, int64_t strideX_mat, int64_t strideX_elem,
                         int32_t *info, cudaStream_t stream);

/* ---------------------------------------------------------------------------------------
 * Batched linear solve with the same factorisation.
 *
 * Solves A_b x_b = y_b for every b: Cholesky per eqs. (5)-(7), P:49-61 (R* b = y by forward
 * substitution, then R x = b), LDL per eqs. (12)-(14), P:87-99 (R* D b = y, then R x = b with
 * R unit upper).  One right-hand side per matrix, as in the paper (x, y in C^{N x 1}).
 *   A: as for the inversion (only the upper triangle and Re a_ii are read; same layouts).
 *   Y, Xv: vector element i of system b at base[b*stride_mat + i*stride_elem]; accepted
 *     layouts: interleaved (stride_mat = 1, stride_elem >= batch) or contiguous
 *     (stride_elem = 1, stride_mat >= n); n = 1: any stride_mat >= 1.  Xv may alias Y with
 *     identical strides; it may not overlap A.
 *   info: as for the inversion; Xv_b is NaN when info[b] != 0.
 * Returns 0, -k for invalid argument k (1-based: 1 batch, 2 n, 3 A, 4/5 A strides, 6 Y,
 * 7/8 Y strides, 9 Xv, 10/11 Xv strides, 12 info), or a cudaError_t from the launch.
 * Asynchronous, stream-ordered; no allocation.  Kernels: one system per thread with the
 * triangle in registers for n <= 8 (c64) / n <= 6 (c128), else one system per CTA. */
int chol_solve_batched_c64(int64_t batch, int n,
                           const cuFloatComplex *A, int64_t strideA_mat, int64_t strideA_elem,
                           const cuFloatComplex *Y, int64_t strideY_mat, int64_t strideY_elem,
                           cuFloatComplex *Xv, int64_t strideX_mat, int64_t strideX_elem,
                           int32_t *info, cudaStream_t stream);
int chol_solve_batched_c128(int64_t batch, int n,
                            const cuDoubleComplex *A, int64_t strideA_mat, int64_t strideA_elem,
                            const cuDoubleComplex *Y, int64_t strideY_mat, int64_t strideY_elem,
                            cuDoubleComplex *Xv, int64_t strideX_mat, int64_t strideX_elem,
                            int32_t *info, cudaStream_t stream);
int ldl_solve_batched_c64(int64_t batch, int n,
                          const cuFloatComplex *A, int64_t strideA_mat, int64_t strideA_elem,
                          const cuFloatComplex *Y, int64_t strideY_mat, int64_t strideY_elem,
                          cuFloatComplex *Xv, int64_t strideX_mat, int64_t strideX_elem,
                          int32_t *info, cudaStream_t stream);
int ldl_solve_batched_c128(int64_t batch, int n,
                           const cuDoubleComplex *A, int64_t strideA_mat, int64_t strideA_elem,
                           const cuDoubleComplex *Y, int64_t strideY_mat, int64_t strideY_elem,
                           cuDoubleComplex *Xv, int64_t strideX_mat, int64_t strideX_elem,
                           int32_t *info, cudaStream_t stream);

/* The batched solve from HOST buffers (end to end): the same chunked, double-buffered
 * H2D -> kernel -> D2H pipeline as hpdinv_inv_host.  A, Y, Xv host pointers with the device
 * entry points' layouts (strides in elements; only the upper triangle of an interleaved A
 * crosses PCIe); d_work / work_bytes: caller-owned device workspace, 256-byte aligned, at least
 * hpdinv_solve_host_workspace_bytes(dtype, n, chunk) (chunk is halved until it fits).
 * Returns 0, -k for invalid argument k (1 method, 2 dtype, 3 batch, 4 n, 5/6 A, 8/9 Y,
 * 11/12 Xv, 14 info, 15 d_work, 16 work_bytes), or a cudaError_t.  Asynchronous on `stream`. */
size_t hpdinv_solve_host_workspace_bytes(int dtype, int n, int64_t chunk);
int hpdinv_solve_host(int method, int dtype, int64_t batch, int n,
                      const void *A_host, int64_t strideA_mat, int64_t strideA_elem,
                      const void *Y_host, int64_t strideY_mat, int64_t strideY_elem,
                      void *X_host, int64_t strideX_mat, int64_t strideX_elem, int32_t *info_host,
                      void *d_work, size_t work_bytes, int64_t chunk, cudaStream_t stream);

/* Name of the solve kernel the dispatcher would launch (static string; NULL if invalid). */
const char *hpdinv_solve_kernel_name(int method, int dtype, int n);

/* ---------------------------------------------------------------------------------------
 * The paper's existing inversion methods on the GPU, for measuring the
 * Table 1 comparison on B200.  All start from the Cholesky factor (eqs. 3-4):
 *   method 0 / 1: the proposed method (Cholesky / LDL) -- exactly chol_/ldl_inv_batched_*;
 *   method 2: equation solving, eq. (15), P:103-113 (R* b_i = e_i, then R x_i = b_i);
 *   method 3: triangular matrix operations, eqs. (16)-(19), P:115-133 (M = R^-1, X = M M*).
 * dtype 0 = complex64, 1 = complex128.  Arguments 3..12 and the contract (layouts, info, NaN
 * fill, mirror, stream order, no allocation) are those of chol_inv_batched_*; returns 0, -k for
 * invalid argument k (1 method, 2 dtype, 3 batch, 4 n, 5 A, ...), or a cudaError_t.  Methods
 * 2 and 3: one matrix per thread in registers for n <= 8 (c64) / n <= 6 (c128), otherwise one
 * matrix per CTA (correctness path). */
int hpdinv_inv_batched_method(int method, int dtype, int64_t batch, int n,
                              const void *A, int64_t strideA_mat, int64_t strideA_elem,
                              void *X, int64_t strideX_mat, int64_t strideX_elem,
                              int32_t *info, cudaStream_t stream);

/* Kernel a method-2/3 call would launch (static string; NULL for methods 0/1 or bad args). */
const char *hpdinv_method_kernel_name(int method, int dtype, int n);

/* ---------------------------------------------------------------------------------------
 * Non-Hermitian inversion through the HPD path: for an
 * arbitrary nonsingular D, A = D D* is HPD; X = A^-1 by Cholesky (eqs. 3-4) + the proposed
 * inversion (eqs. 20-24); D^-1 = D* X.  Fused in one launch (D read, D^-1 written).
 *   D, Dinv: element (i,j) of matrix b at base[b*stride_mat + (i*n+j)*stride_elem] (ALL n^2
 *     entries of D are read); layouts and argument numbering as chol_inv_batched_*; Dinv may
 *     not overlap D.
 *   info[b]: the Cholesky info of A_b = D_b D_b* (0 <=> numerically nonsingular); Dinv_b is
 *     NaN when info[b] != 0.
 * Kernels: one matrix per thread in registers for n <= 8 (c64) / n <= 6 (c128), otherwise one
 * matrix per CTA. */
int nonherm_inv_batched_c64(int64_t batch, int n,
                            const cuFloatComplex *D, int64_t strideD_mat, int64_t strideD_elem,
                            cuFloatComplex *Dinv, int64_t strideX_mat, int64_t strideX_elem,
                            int32_t *info, cudaStream_t stream);
int nonherm_inv_batched_c128(int64_t batch, int n,
                             const cuDoubleComplex *D, int64_t strideD_mat, int64_t strideD_elem,
                             cuDoubleComplex *Dinv, int64_t strideX_mat, int64_t strideX_elem,
                             int32_t *info, cudaStream_t stream);

/* Kernel the non-Hermitian entry point launches (static string; NULL if invalid). */
const char *hpdinv_nonherm_kernel_name(int dtype, int n);

/* ---------------------------------------------------------------------------------------
 * Fixed-point (Q-format) emulation of the inversion methods for the paper's accuracy study
 * (§IV.C, Fig. 1).  The paper fixes no format; the arithmetic
 * is DESIGN.md's reading F1-F7 (Q(m, f) raws, saturation, one round-half-even per F4 product
 * component, round-half-even division by the pivot, exact rounded square root, term-by-term
 * accumulation).  method: 0 proposed (Cholesky + eqs. 20-24), 1 equation solving (eq. 15),
 * 2 triangular matrix operations (eqs. 16-19).
 *   A, X: device, contiguous batch x n x n, each complex entry an interleaved (re, im) pair of
 *     int64 raws (value = raw * 2^-f); only the upper triangle and Re a_ii of A are read; X is
 *     written in full (Hermitian mirror) and is zero when info != 0.
 *   info[b]: first 1-based pivot with a non-positive radicand, else 0; nsat[b]: number of
 *     saturation events in matrix b (int64).
 * 1 <= m, 1 <= f, m + f <= 40; 1 <= n <= 16.  Returns 0, -k for invalid argument k (1 method,
 * 2 the format (m, f), 4 batch, 5 n, 6 A, 7 X, 8 info, 9 nsat), or a cudaError_t.
 * One matrix per thread, integer ALU; asynchronous, stream-ordered, no allocation. */
int hpdinv_fxp_inv_batched(int method, int m, int f, int64_t batch, int n, const int64_t *A,
                           int64_t *X, int32_t *info, int64_t *nsat, cudaStream_t stream);

/* ---------------------------------------------------------------------------------------
 * Host-buffer entry point (end-to-end use from host memory).
 *
 * hpdinv_inv_host runs the same hot path on matrices that live in HOST memory (pinned
 * memory recommended; pageable memory works but serialises the copies): the batch is cut
 * into chunks of `chunk` matrices (0 = automatic) that flow through a double-buffered
 * H2D -> kernel -> D2H pipeline on two internal copy streams plus `stream` for the kernels.
 * Only the upper triangle is copied host->device for an interleaved (SoA) host A.
 *   method: 0 Cholesky, 1 LDL, 2 the non-Hermitian inversion of nonherm_inv_batched_* (all n^2
 *   entries of A are copied; half a slot each for input and output).  dtype: 0 complex64,
 *   1 complex128.
 *   A_host / X_host / info_host: host pointers, same addressing and layout classes as the
 *   device entry points (strides in elements).  X_host may not alias A_host.
 *   d_work / work_bytes: caller-owned device workspace, 256-byte aligned, at least
 *   hpdinv_host_workspace_bytes(dtype, n, chunk) bytes (chunk is halved until it fits).
 * Asynchronous and stream-ordered like cudaMemcpyAsync: the call returns once everything
 * is enqueued; X_host / info_host are valid when `stream` reaches the point of the call.
 * Returns 0, -k for invalid argument k (1-based), or a cudaError_t. */
size_t hpdinv_host_workspace_bytes(int dtype, int n, int64_t chunk);

int hpdinv_inv_host(int method, int dtype, int64_t batch, int n,
                    const void *A_host, int64_t strideA_mat, int64_t strideA_elem,
                    void *X_host, int64_t strideX_mat, int64_t strideX_elem,
                    int32_t *info_host, void *d_work, size_t work_bytes, int64_t chunk,
                    cudaStream_t stream);

/* Name of the kernel the dispatcher would launch for these arguments (for tests/bench
 * evidence); NULL when the arguments are invalid.  method: 0 Cholesky, 1 LDL;
 * dtype: 0 c64, 1 c128.  The string is static. */
const char *hpdinv_kernel_name(int method, int dtype, int64_t batch, int n,
                               int64_t strideA_mat, int64_t strideA_elem,
                               int64_t strideX_mat, int64_t strideX_elem);

/* Library version string (static). */
const char *hpdinv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HPDINV_H */
