"""Shared helpers for the -m gpu parity tests (CUDA path vs the fp64 oracle)."""
import numpy as np
import torch

import oracle
import paper_1111_4144_b200 as hp
from paper_1111_4144_b200 import workloads as wl

# Tolerances (BASELINE.json north_star, reading R13): per matrix b,
#   max_ij |x_gpu - x_oracle| / max_ij |x_oracle|  <=  TOL * cond_2(A_b)
TOL = {torch.complex64: 2e-5, torch.complex128: 1e-12}


def to_host_c128(A: torch.Tensor) -> np.ndarray:
    """Exact upcast of the device input bits to complex128 (contiguous (batch, n, n))."""
    return A.detach().contiguous().cpu().to(torch.complex128).numpy()


def cond2(Ah: np.ndarray) -> np.ndarray:
    w = np.linalg.eigvalsh(Ah)        # reads the lower triangle; A is exactly Hermitian
    return w[:, -1] / w[:, 0]


def compare(X_gpu: np.ndarray, X_or: np.ndarray, info_gpu, info_or, cond, tol):
    """Returns the max of err_b / cond_b over matrices; asserts info bit-exactness."""
    info_gpu = np.asarray(info_gpu)
    info_or = np.asarray(info_or)
    assert np.array_equal(info_gpu, info_or), "info mismatch at %s" % np.nonzero(info_gpu != info_or)[0][:10]
    ok = info_or == 0
    if not ok.any():
        return 0.0
    d = np.abs(X_gpu[ok] - X_or[ok]).reshape(ok.sum(), -1).max(axis=1)
    s = np.abs(X_or[ok]).reshape(ok.sum(), -1).max(axis=1)
    ratio = d / s / cond[ok]
    worst = int(np.argmax(ratio))
    assert ratio[worst] <= tol, "err/cond %.3e > %.1e at matrix %d" % (ratio[worst], tol, np.nonzero(ok)[0][worst])
    return float(ratio.max())


def check_mirror(X: np.ndarray, info: np.ndarray):
    ok = np.asarray(info) == 0
    Xo = X[ok]
    assert np.array_equal(Xo, np.conj(np.transpose(Xo, (0, 2, 1)))), "mirror not bit-exact"
    d = np.diagonal(Xo, axis1=1, axis2=2)
    assert np.all(d.imag == 0) and not np.signbit(d.imag).any(), "Im x_ii must be +0"
    if (~ok).any():
        assert np.isnan(X[~ok]).all(), "flagged matrices must be NaN-filled"


def run_gpu(A_dev: torch.Tensor, method: str, layout: str, ld=None, x_layout=None):
    """Lay A out, run the library, return (X contiguous host complex128, info host, X view)."""
    _, view = wl.to_layout(A_dev, layout, ld)
    if x_layout is None or x_layout == layout:
        X = wl.empty_like_layout(view)
    else:
        _, X = wl.to_layout(torch.zeros_like(A_dev), x_layout)
    X, info = hp.invert(view, method, X=X)
    torch.cuda.synchronize()
    return X.contiguous().cpu().to(torch.complex128).numpy(), info.cpu().numpy(), X


def oracle_run(Ah: np.ndarray, method: str):
    return oracle.inv_batched(Ah, method)
