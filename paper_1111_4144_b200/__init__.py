"""paper_1111_4144_b200 -- B200-native batched inversion of small complex HPD matrices.

Thin Python binding over the C ABI of ``include/hpdinv.h`` (libhpdinv.so): argument
marshalling only -- every step of the path (load, Cholesky / LDL, the paper's direct
inversion, mirror, store) runs in the library's sm_100a kernels.

Tensors are (batch, n, n) views whose element (i, j) of matrix b is at
``data[b*stride_mat + (i*n + j)*stride_elem]`` -- a contiguous tensor is the AoS layout,
``workloads.soa_view`` builds the interleaved (SoA) layout.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Tuple

import torch

from ._lib import EXPORTS, HpdinvError, lib  # noqa: F401

__all__ = [
    "chol_inv_batched_c64", "chol_inv_batched_c128", "ldl_inv_batched_c64",
    "ldl_inv_batched_c128", "chol_solve_batched_c64", "chol_solve_batched_c128",
    "ldl_solve_batched_c64", "ldl_solve_batched_c128", "solve", "solve_host", "solve_host_workspace_bytes",
    "solve_kernel_name", "invert",
    "invert_method", "method_kernel_name", "nonherm_inv_batched_c64", "nonherm_inv_batched_c128",
    "invert_nonhermitian", "nonherm_kernel_name", "fxp_invert", "invert_host", "host_workspace_bytes", "kernel_name", "version", "HpdinvError",
]


def _strides(t: torch.Tensor) -> Tuple[int, int]:
    if t.dim() != 3 or t.shape[1] != t.shape[2]:
        raise ValueError("expected a (batch, n, n) tensor, got shape %s" % (tuple(t.shape),))
    n = t.shape[1]
    s0, s1, s2 = t.stride()
    if n > 1 and s1 != n * s2:
        raise ValueError("unsupported strides %s: need stride(1) == n*stride(2)" % (t.stride(),))
    return s0, s2


_WORKSPACES = {}


def _auto_workspace(nbytes: int) -> torch.Tensor:
    """Device workspace for the host entry points when the caller passes none.  It is kept
    (per device, grown on demand) rather than freed on return: the copies the call enqueued on
    the library's internal streams still use it, and those streams are invisible to PyTorch's
    caching allocator."""
    dev = torch.cuda.current_device()
    ws = _WORKSPACES.get(dev)
    if ws is None or ws.numel() < nbytes:
        if ws is not None:
            torch.cuda.synchronize(dev)          # the old buffer may still be in flight
        ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        _WORKSPACES[dev] = ws
    return ws


def _stream_handle(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _call(fname: str, dtype: torch.dtype, A: torch.Tensor, X: Optional[torch.Tensor],
          info: Optional[torch.Tensor], stream) -> Tuple[torch.Tensor, torch.Tensor]:
    if A.dtype != dtype:
        raise TypeError("%s expects %s, got %s" % (fname, dtype, A.dtype))
    if not A.is_cuda:
        raise ValueError("%s: A must be a CUDA tensor (no CPU path exists)" % fname)
    batch, n = A.shape[0], A.shape[1]
    sAm, sAe = _strides(A)
    if X is None:
        X = torch.empty_strided(A.shape, A.stride(), dtype=dtype, device=A.device)
    sXm, sXe = _strides(X)
    if info is None:
        info = torch.empty(batch, dtype=torch.int32, device=A.device)
    if info.dtype != torch.int32 or info.numel() < batch or not info.is_contiguous():
        raise ValueError("info must be a contiguous int32 tensor of length >= batch")
    rc = getattr(lib(), fname)(batch, n, ctypes.c_void_p(A.data_ptr()), sAm, sAe,
                               ctypes.c_void_p(X.data_ptr()), sXm, sXe,
                               ctypes.c_void_p(info.data_ptr()), ctypes.c_void_p(_stream_handle(stream)))
    if rc < 0:
        raise ValueError("%s rejected argument %d" % (fname, -rc))
    if rc > 0:
        raise HpdinvError("%s: CUDA error %d at launch" % (fname, rc))
    return X, info


def chol_inv_batched_c64(A, X=None, info=None, stream=None):
    """Cholesky (eqs. 3-4) + proposed inversion (eqs. 20-24) + mirror, complex64."""
    return _call("chol_inv_batched_c64", torch.complex64, A, X, info, stream)


def chol_inv_batched_c128(A, X=None, info=None, stream=None):
    """Cholesky (eqs. 3-4) + proposed inversion (eqs. 20-24) + mirror, complex128."""
    return _call("chol_inv_batched_c128", torch.complex128, A, X, info, stream)


def ldl_inv_batched_c64(A, X=None, info=None, stream=None):
    """LDL (eqs. 10-11) + proposed inversion (eqs. 25-29) + mirror, complex64."""
    return _call("ldl_inv_batched_c64", torch.complex64, A, X, info, stream)


def ldl_inv_batched_c128(A, X=None, info=None, stream=None):
    """LDL (eqs. 10-11) + proposed inversion (eqs. 25-29) + mirror, complex128."""
    return _call("ldl_inv_batched_c128", torch.complex128, A, X, info, stream)


_DISPATCH = {
    ("chol", torch.complex64): chol_inv_batched_c64,
    ("chol", torch.complex128): chol_inv_batched_c128,
    ("ldl", torch.complex64): ldl_inv_batched_c64,
    ("ldl", torch.complex128): ldl_inv_batched_c128,
}


def invert(A, method: str = "chol", X=None, info=None, stream=None):
    """Dispatch on (method, A.dtype) to the matching C entry point."""
    return _DISPATCH[(method, A.dtype)](A, X, info, stream)


def _vstrides(v: torch.Tensor) -> Tuple[int, int]:
    if v.dim() != 2:
        raise ValueError("expected a (batch, n) tensor, got shape %s" % (tuple(v.shape),))
    return v.stride(0), v.stride(1)


def _call_solve(fname: str, dtype: torch.dtype, A, Y, Xv, info, stream):
    for t, nm in ((A, "A"), (Y, "Y")):
        if t.dtype != dtype:
            raise TypeError("%s expects %s for %s, got %s" % (fname, dtype, nm, t.dtype))
        if not t.is_cuda:
            raise ValueError("%s: %s must be a CUDA tensor (no CPU path exists)" % (fname, nm))
    batch, n = A.shape[0], A.shape[1]
    if tuple(Y.shape) != (batch, n):
        raise ValueError("Y must have shape (batch, n)")
    sAm, sAe = _strides(A)
    sYm, sYe = _vstrides(Y)
    if Xv is None:
        Xv = torch.empty_strided(Y.shape, Y.stride(), dtype=dtype, device=Y.device)
    sXm, sXe = _vstrides(Xv)
    if info is None:
        info = torch.empty(batch, dtype=torch.int32, device=A.device)
    if info.dtype != torch.int32 or info.numel() < batch or not info.is_contiguous():
        raise ValueError("info must be a contiguous int32 tensor of length >= batch")
    rc = getattr(lib(), fname)(batch, n, ctypes.c_void_p(A.data_ptr()), sAm, sAe,
                               ctypes.c_void_p(Y.data_ptr()), sYm, sYe,
                               ctypes.c_void_p(Xv.data_ptr()), sXm, sXe,
                               ctypes.c_void_p(info.data_ptr()), ctypes.c_void_p(_stream_handle(stream)))
    if rc < 0:
        raise ValueError("%s rejected argument %d" % (fname, -rc))
    if rc > 0:
        raise HpdinvError("%s: CUDA error %d at launch" % (fname, rc))
    return Xv, info


def chol_solve_batched_c64(A, Y, Xv=None, info=None, stream=None):
    """A x = y by Cholesky, eqs. (5)-(7), complex64.  Y, Xv: (batch, n) views."""
    return _call_solve("chol_solve_batched_c64", torch.complex64, A, Y, Xv, info, stream)


def chol_solve_batched_c128(A, Y, Xv=None, info=None, stream=None):
    """A x = y by Cholesky, eqs. (5)-(7), complex128."""
    return _call_solve("chol_solve_batched_c128", torch.complex128, A, Y, Xv, info, stream)


def ldl_solve_batched_c64(A, Y, Xv=None, info=None, stream=None):
    """A x = y by LDL, eqs. (12)-(14), complex64."""
    return _call_solve("ldl_solve_batched_c64", torch.complex64, A, Y, Xv, info, stream)


def ldl_solve_batched_c128(A, Y, Xv=None, info=None, stream=None):
    """A x = y by LDL, eqs. (12)-(14), complex128."""
    return _call_solve("ldl_solve_batched_c128", torch.complex128, A, Y, Xv, info, stream)


_SOLVE = {
    ("chol", torch.complex64): chol_solve_batched_c64,
    ("chol", torch.complex128): chol_solve_batched_c128,
    ("ldl", torch.complex64): ldl_solve_batched_c64,
    ("ldl", torch.complex128): ldl_solve_batched_c128,
}


def solve(A, Y, method: str = "chol", Xv=None, info=None, stream=None):
    """Batched A_b x_b = y_b with the same factorisation."""
    return _SOLVE[(method, A.dtype)](A, Y, Xv, info, stream)


def solve_host(A_host: torch.Tensor, Y_host: torch.Tensor, method: str = "chol", X_host=None, info_host=None,
               workspace: Optional[torch.Tensor] = None, chunk: int = 0, stream=None):
    """hpdinv_solve_host: the batched solve from host (pinned) tensors, end to end."""
    if A_host.is_cuda or Y_host.is_cuda:
        raise ValueError("solve_host expects host tensors")
    dtype = A_host.dtype
    batch, n = A_host.shape[0], A_host.shape[1]
    sAm, sAe = _strides(A_host)
    sYm, sYe = _vstrides(Y_host)
    if X_host is None:
        X_host = torch.empty_strided(Y_host.shape, Y_host.stride(), dtype=dtype, pin_memory=True)
    sXm, sXe = _vstrides(X_host)
    if info_host is None:
        info_host = torch.empty(batch, dtype=torch.int32, pin_memory=True)
    dt = {torch.complex64: 0, torch.complex128: 1}[dtype]
    if workspace is None:
        ch = chunk if chunk > 0 else max(min(batch, 4096), (batch + 7) // 8)
        workspace = _auto_workspace(int(lib().hpdinv_solve_host_workspace_bytes(dt, n, ch)))
    rc = lib().hpdinv_solve_host({"chol": 0, "ldl": 1}[method], dt, batch, n,
                                 ctypes.c_void_p(A_host.data_ptr()), sAm, sAe,
                                 ctypes.c_void_p(Y_host.data_ptr()), sYm, sYe,
                                 ctypes.c_void_p(X_host.data_ptr()), sXm, sXe,
                                 ctypes.c_void_p(info_host.data_ptr()), ctypes.c_void_p(workspace.data_ptr()),
                                 workspace.numel(), chunk, ctypes.c_void_p(_stream_handle(stream)))
    if rc < 0:
        raise ValueError("hpdinv_solve_host rejected argument %d" % (-rc))
    if rc > 0:
        raise HpdinvError("hpdinv_solve_host: CUDA error %d" % rc)
    return X_host, info_host


def solve_host_workspace_bytes(dtype: torch.dtype, n: int, chunk: int) -> int:
    return int(lib().hpdinv_solve_host_workspace_bytes({torch.complex64: 0, torch.complex128: 1}[dtype], n, chunk))


def solve_kernel_name(method: str, dtype: torch.dtype, n: int):
    r = lib().hpdinv_solve_kernel_name({"chol": 0, "ldl": 1}[method], {torch.complex64: 0, torch.complex128: 1}[dtype], n)
    return r.decode() if r else None


def nonherm_inv_batched_c64(D, Dinv=None, info=None, stream=None):
    """D^-1 = D* (D D*)^-1 via Cholesky + the proposed inversion, complex64."""
    return _call("nonherm_inv_batched_c64", torch.complex64, D, Dinv, info, stream)


def nonherm_inv_batched_c128(D, Dinv=None, info=None, stream=None):
    """D^-1 = D* (D D*)^-1 via Cholesky + the proposed inversion, complex128."""
    return _call("nonherm_inv_batched_c128", torch.complex128, D, Dinv, info, stream)


def invert_nonhermitian(D, Dinv=None, info=None, stream=None):
    """Batched inverse of arbitrary (non-Hermitian) matrices."""
    f = nonherm_inv_batched_c64 if D.dtype == torch.complex64 else nonherm_inv_batched_c128
    return f(D, Dinv, info, stream)


def nonherm_kernel_name(dtype: torch.dtype, n: int):
    r = lib().hpdinv_nonherm_kernel_name({torch.complex64: 0, torch.complex128: 1}[dtype], n)
    return r.decode() if r else None


FXP_METHODS = {"proposed": 0, "eqsolve": 1, "trimat": 2}


def fxp_invert(A_raw: torch.Tensor, m: int, f: int, method: str = "proposed", X=None, info=None,
               nsat=None, stream=None):
    """Fixed-point Q(m, f) emulation on the GPU: A_raw is a contiguous CUDA
    int64 tensor (batch, n, n, 2) of raws.  Returns (X_raw, info, nsat)."""
    if A_raw.dtype != torch.int64 or not A_raw.is_cuda or not A_raw.is_contiguous():
        raise ValueError("fxp_invert: A_raw must be a contiguous CUDA int64 tensor (batch, n, n, 2)")
    batch, n = A_raw.shape[0], A_raw.shape[1]
    X = torch.empty_like(A_raw) if X is None else X
    info = torch.empty(batch, dtype=torch.int32, device=A_raw.device) if info is None else info
    nsat = torch.empty(batch, dtype=torch.int64, device=A_raw.device) if nsat is None else nsat
    rc = lib().hpdinv_fxp_inv_batched(FXP_METHODS[method], m, f, batch, n, ctypes.c_void_p(A_raw.data_ptr()),
                                      ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(info.data_ptr()),
                                      ctypes.c_void_p(nsat.data_ptr()), ctypes.c_void_p(_stream_handle(stream)))
    if rc < 0:
        raise ValueError("hpdinv_fxp_inv_batched rejected argument %d" % (-rc))
    if rc > 0:
        raise HpdinvError("hpdinv_fxp_inv_batched: CUDA error %d at launch" % rc)
    return X, info, nsat


METHOD_IDS = {"chol": 0, "ldl": 1, "eqsolve": 2, "trimat": 3}


def invert_method(A, method: str, X=None, info=None, stream=None):
    """hpdinv_inv_batched_method: the paper's existing methods on the GPU --
    "eqsolve" (eq. 15) and "trimat" (eqs. 16-19) -- or the proposed "chol" / "ldl"."""
    dtype = {torch.complex64: 0, torch.complex128: 1}[A.dtype]
    if not A.is_cuda:
        raise ValueError("invert_method: A must be a CUDA tensor (no CPU path exists)")
    batch, n = A.shape[0], A.shape[1]
    sAm, sAe = _strides(A)
    if X is None:
        X = torch.empty_strided(A.shape, A.stride(), dtype=A.dtype, device=A.device)
    sXm, sXe = _strides(X)
    if info is None:
        info = torch.empty(batch, dtype=torch.int32, device=A.device)
    rc = lib().hpdinv_inv_batched_method(METHOD_IDS[method], dtype, batch, n, ctypes.c_void_p(A.data_ptr()),
                                         sAm, sAe, ctypes.c_void_p(X.data_ptr()), sXm, sXe,
                                         ctypes.c_void_p(info.data_ptr()), ctypes.c_void_p(_stream_handle(stream)))
    if rc < 0:
        raise ValueError("hpdinv_inv_batched_method rejected argument %d" % (-rc))
    if rc > 0:
        raise HpdinvError("hpdinv_inv_batched_method: CUDA error %d at launch" % rc)
    return X, info


def method_kernel_name(method: str, dtype: torch.dtype, n: int):
    r = lib().hpdinv_method_kernel_name(METHOD_IDS[method], {torch.complex64: 0, torch.complex128: 1}[dtype], n)
    return r.decode() if r else None


def host_workspace_bytes(dtype: torch.dtype, n: int, chunk: int) -> int:
    return int(lib().hpdinv_host_workspace_bytes({torch.complex64: 0, torch.complex128: 1}[dtype], n, chunk))


def invert_host(A_host: torch.Tensor, method: str = "chol", X_host=None, info_host=None,
                workspace: Optional[torch.Tensor] = None, chunk: int = 0, stream=None):
    """hpdinv_inv_host: A_host / X_host / info_host are CPU tensors (pin them for overlap);
    `workspace` is a CUDA uint8 tensor.  Asynchronous on `stream` (synchronize before
    reading X_host)."""
    if A_host.is_cuda:
        raise ValueError("invert_host expects host tensors")
    dtype = A_host.dtype
    batch, n = A_host.shape[0], A_host.shape[1]
    sAm, sAe = _strides(A_host)
    if X_host is None:
        X_host = torch.empty_strided(A_host.shape, A_host.stride(), dtype=dtype, pin_memory=True)
    sXm, sXe = _strides(X_host)
    if info_host is None:
        info_host = torch.empty(batch, dtype=torch.int32, pin_memory=True)
    if workspace is None:
        ch = chunk if chunk > 0 else max(min(batch, 4096), (batch + 7) // 8)
        workspace = _auto_workspace(host_workspace_bytes(dtype, n, ch))
    rc = lib().hpdinv_inv_host({"chol": 0, "ldl": 1, "nonherm": 2}[method], {torch.complex64: 0, torch.complex128: 1}[dtype],
                               batch, n, ctypes.c_void_p(A_host.data_ptr()), sAm, sAe,
                               ctypes.c_void_p(X_host.data_ptr()), sXm, sXe,
                               ctypes.c_void_p(info_host.data_ptr()), ctypes.c_void_p(workspace.data_ptr()),
                               workspace.numel(), chunk, ctypes.c_void_p(_stream_handle(stream)))
    if rc < 0:
        raise ValueError("hpdinv_inv_host rejected argument %d" % (-rc))
    if rc > 0:
        raise HpdinvError("hpdinv_inv_host: CUDA error %d" % rc)
    return X_host, info_host


def kernel_name(method: str, dtype: torch.dtype, batch: int, n: int, sA=(None, None), sX=(None, None)):
    """Name of the kernel the library's dispatcher selects for these arguments."""
    sAm, sAe = sA if sA[0] is not None else (n * n, 1)
    sXm, sXe = sX if sX[0] is not None else (sAm, sAe)
    r = lib().hpdinv_kernel_name({"chol": 0, "ldl": 1}[method],
                                 {torch.complex64: 0, torch.complex128: 1}[dtype],
                                 batch, n, sAm, sAe, sXm, sXe)
    return r.decode() if r else None


def version() -> str:
    return lib().hpdinv_version().decode()
