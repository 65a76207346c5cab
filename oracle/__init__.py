"""fp64 CPU oracle for batched HPD inversion (arxiv/paper_1111_4144) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1111_4144_b200``) never imports it, and the two share no code: this is a ctypes
wrapper around ``hpdinv_oracle.c`` (plain C99 complex loops that follow PAPER.md's equations
in order; see that file for the per-function citations).

Parity status: every function here is pinned by ``tests/test_oracle_pins.py``
and ``tests/test_counts.py`` against closed forms, exact-integer families, exact rational
Gauss-Jordan, LAPACK and the paper's Table 1 counts -- except the fixed-point study of
§IV.C (Fig. 1), which is out of scope and "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hpdinv_oracle.c")
_HDR = os.path.join(_HERE, "hpdinv_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_FXP_SRC = os.path.join(_HERE, "fxp_oracle.c")      # fixed-point emulation
_FXP_HDR = os.path.join(_HERE, "fxp_oracle.h")

PAPER_CONVENTION = 0
FULL_EXPLOITATION = 1

METHODS = {"chol": 0, "ldl": 1, "eqsolve": 2, "trimat": 3}


class Counts(ctypes.Structure):
    _fields_ = [("cmul", ctypes.c_longlong), ("cdiv", ctypes.c_longlong),
                ("cadd", ctypes.c_longlong), ("csqrt", ctypes.c_longlong)]

    def as_dict(self) -> Dict[str, int]:
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


def build(force: bool = False) -> str:
    """Compile ``liboracle.so`` with gcc (plain -O2, OpenMP across matrices only)."""
    newest = max(os.path.getmtime(p) for p in (_SRC, _HDR, _FXP_SRC, _FXP_HDR))
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= newest:
        return _LIB
    tmp = _LIB + ".tmp%d" % os.getpid()
    cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
           "-o", tmp, _SRC, _FXP_SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I = ctypes.c_int
        I64 = ctypes.c_int64
        CP = ctypes.POINTER(Counts)
        sig = {
            "oracle_chol_upper": (I, [I, P, P, CP]),
            "oracle_ldl_upper": (I, [I, P, P, P, CP]),
            "oracle_proposed_inv_chol": (None, [I, P, P, CP]),
            "oracle_proposed_inv_ldl": (None, [I, P, P, P, CP]),
            "oracle_mirror": (None, [I, P]),
            "oracle_eqsolve_inv": (None, [I, P, P, I, CP]),
            "oracle_trimat_inv": (None, [I, P, P, I, CP]),
            "oracle_solve_chol": (None, [I, P, P, P, CP]),
            "oracle_solve_ldl": (None, [I, P, P, P, P, CP]),
            "oracle_nonhermitian_inv": (I, [I, P, P]),
            "oracle_inv_batched": (I, [I64, I, P, I64, I64, P, I64, I64, P, I, I]),
            "oracle_solve_batched": (I, [I64, I, P, I64, I64, P, P, P, I, I]),
            "oracle_nonherm_batched": (I, [I64, I, P, P, P, I]),
            "oracle_max_threads": (I, []),
            "oracle_fxp_inv_batched": (I, [I64, I, P, P, P, P, I, I, I, I]),
            "oracle_fxp_op": (I, [I, I, I, I64, I64, I64, I64, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _ptr(a: np.ndarray) -> int:
    return a.__array_interface__["data"][0]


def _counts(count: bool):
    return Counts() if count else None


def _cref(c):
    return ctypes.byref(c) if c is not None else None


# ------------------------------------------------------------------ single-matrix routines
def chol_upper(A, count: bool = False):
    """Eqs. (3)-(4): returns (R, info[, counts])."""
    A = _c128(A)
    n = A.shape[0]
    R = np.zeros((n, n), np.complex128)
    c = _counts(count)
    info = lib().oracle_chol_upper(n, _ptr(A), _ptr(R), _cref(c))
    return (R, info, c.as_dict()) if count else (R, info)


def ldl_upper(A, count: bool = False):
    """Eqs. (10)-(11): returns (R, d, info[, counts])."""
    A = _c128(A)
    n = A.shape[0]
    R = np.zeros((n, n), np.complex128)
    d = np.zeros(n, np.float64)
    c = _counts(count)
    info = lib().oracle_ldl_upper(n, _ptr(A), _ptr(R), _ptr(d), _cref(c))
    return (R, d, info, c.as_dict()) if count else (R, d, info)


def proposed_inv_chol(R, count: bool = False):
    """Eqs. (20)-(24) + mirror."""
    R = _c128(R)
    n = R.shape[0]
    X = np.zeros((n, n), np.complex128)
    c = _counts(count)
    lib().oracle_proposed_inv_chol(n, _ptr(R), _ptr(X), _cref(c))
    return (X, c.as_dict()) if count else X


def proposed_inv_ldl(R, d, count: bool = False):
    """Eqs. (25)-(29) + mirror."""
    R = _c128(R)
    d = np.ascontiguousarray(np.asarray(d, np.float64))
    n = R.shape[0]
    X = np.zeros((n, n), np.complex128)
    c = _counts(count)
    lib().oracle_proposed_inv_ldl(n, _ptr(R), _ptr(d), _ptr(X), _cref(c))
    return (X, c.as_dict()) if count else X


def mirror(X):
    X = _c128(X).copy()
    lib().oracle_mirror(X.shape[0], _ptr(X))
    return X


def eqsolve_inv(R, convention: int = PAPER_CONVENTION, count: bool = False):
    """Eq. (15) via eqs. (6)-(7)."""
    R = _c128(R)
    n = R.shape[0]
    X = np.zeros((n, n), np.complex128)
    c = _counts(count)
    lib().oracle_eqsolve_inv(n, _ptr(R), _ptr(X), convention, _cref(c))
    return (X, c.as_dict()) if count else X


def trimat_inv(R, convention: int = PAPER_CONVENTION, count: bool = False):
    """Eqs. (16)-(19)."""
    R = _c128(R)
    n = R.shape[0]
    X = np.zeros((n, n), np.complex128)
    c = _counts(count)
    lib().oracle_trimat_inv(n, _ptr(R), _ptr(X), convention, _cref(c))
    return (X, c.as_dict()) if count else X


def solve_chol(R, y, count: bool = False):
    """Eqs. (5)-(7)."""
    R = _c128(R)
    y = _c128(y)
    x = np.zeros_like(y)
    c = _counts(count)
    lib().oracle_solve_chol(R.shape[0], _ptr(R), _ptr(y), _ptr(x), _cref(c))
    return (x, c.as_dict()) if count else x


def solve_ldl(R, d, y, count: bool = False):
    """Eqs. (12)-(14)."""
    R = _c128(R)
    d = np.ascontiguousarray(np.asarray(d, np.float64))
    y = _c128(y)
    x = np.zeros_like(y)
    c = _counts(count)
    lib().oracle_solve_ldl(R.shape[0], _ptr(R), _ptr(d), _ptr(y), _ptr(x), _cref(c))
    return (x, c.as_dict()) if count else x


def nonhermitian_inv(D) -> Tuple[np.ndarray, int]:
    """D^-1 = D* (DD*)^-1."""
    D = _c128(D)
    n = D.shape[0]
    Di = np.zeros((n, n), np.complex128)
    info = lib().oracle_nonhermitian_inv(n, _ptr(D), _ptr(Di))
    return Di, info


# ------------------------------------------------------------------------------ batched
def _mat_strides(A: np.ndarray) -> Tuple[int, int]:
    """(stride_mat, stride_elem) in elements for a (batch, n, n) complex128 view."""
    if A.dtype != np.complex128 or A.ndim != 3 or A.shape[1] != A.shape[2]:
        raise ValueError("expected a (batch, n, n) complex128 array")
    n = A.shape[1]
    s0, s1, s2 = (s // 16 for s in A.strides)
    if any(s % 16 for s in A.strides) or s1 != n * s2:
        raise ValueError("unsupported strides %r" % (A.strides,))
    return s0, s2


def inv_batched(A: np.ndarray, method: str = "chol", nthreads: int = 0):
    """Batched inversion of a (batch, n, n) complex128 view (any strides of the form
    base[b*sm + (i*n+j)*se]).  Returns (X contiguous (batch, n, n), info int32[batch])."""
    batch, n = A.shape[0], A.shape[1]
    sm, se = _mat_strides(A)
    X = np.empty((batch, n, n), np.complex128)
    info = np.zeros(batch, np.int32)
    rc = lib().oracle_inv_batched(batch, n, _ptr(A), sm, se, _ptr(X), n * n, 1, _ptr(info),
                                  METHODS[method], int(nthreads))
    if rc != 0:
        raise ValueError("oracle_inv_batched rejected its arguments (rc=%d)" % rc)
    return X, info


def solve_batched(A: np.ndarray, y: np.ndarray, method: str = "chol", nthreads: int = 0):
    """Batched linear solve A_b x_b = y_b (eqs. 5-7 / 12-14).  y: (batch, n)."""
    batch, n = A.shape[0], A.shape[1]
    sm, se = _mat_strides(A)
    y = _c128(y).reshape(batch, n)
    x = np.empty((batch, n), np.complex128)
    info = np.zeros(batch, np.int32)
    rc = lib().oracle_solve_batched(batch, n, _ptr(A), sm, se, _ptr(y), _ptr(x), _ptr(info),
                                    {"chol": 0, "ldl": 1}[method], int(nthreads))
    if rc != 0:
        raise ValueError("oracle_solve_batched rejected its arguments (rc=%d)" % rc)
    return x, info


def nonherm_batched(D: np.ndarray, nthreads: int = 0):
    """Batched D^-1 = D* (D D*)^-1.  D: (batch, n, n)."""
    D = np.ascontiguousarray(_c128(D))
    batch, n = D.shape[0], D.shape[1]
    Dinv = np.empty_like(D)
    info = np.zeros(batch, np.int32)
    rc = lib().oracle_nonherm_batched(batch, n, _ptr(D), _ptr(Dinv), _ptr(info), int(nthreads))
    if rc != 0:
        raise ValueError("oracle_nonherm_batched rejected its arguments (rc=%d)" % rc)
    return Dinv, info


FXP_METHODS = {"proposed": 0, "eqsolve": 1, "trimat": 2}


def fxp_inv_batched(A_raw: np.ndarray, m: int, f: int, method: str = "proposed", nthreads: int = 0):
    """Fixed-point Q(m, f) emulation.  A_raw: (batch, n, n, 2) int64 raws.
    Returns (X_raw (batch, n, n, 2) int64, info int32, nsat int64)."""
    A = np.ascontiguousarray(A_raw, dtype=np.int64)
    batch, n = A.shape[0], A.shape[1]
    X = np.zeros_like(A)
    info = np.zeros(batch, np.int32)
    nsat = np.zeros(batch, np.int64)
    rc = lib().oracle_fxp_inv_batched(batch, n, _ptr(A), _ptr(X), _ptr(info), _ptr(nsat), m, f,
                                      FXP_METHODS[method], int(nthreads))
    if rc != 0:
        raise ValueError("oracle_fxp_inv_batched rejected its arguments (rc=%d)" % rc)
    return X, info, nsat


def fxp_op(op: str, m: int, f: int, a, b=(0, 0)):
    """One F4 product ('mul'), F5 quotient ('div', b = (p, 0)) or F6 root ('sqrt') on raws."""
    out = np.zeros(2, np.int64)
    ns = lib().oracle_fxp_op({"mul": 0, "div": 1, "sqrt": 2}[op], m, f, int(a[0]), int(a[1]),
                             int(b[0]), int(b[1]), _ptr(out))
    return (int(out[0]), int(out[1])), int(ns)


def max_threads() -> int:
    return int(lib().oracle_max_threads())
