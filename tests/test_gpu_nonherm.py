"""inversion of non-Hermitian matrices through the HPD path
(A = D D*, X = A^-1 by Cholesky + the proposed inversion, D^-1 = D* X) vs the fp64
oracle (oracle_nonhermitian_inv) on the same seeded inputs; exactly invertible Gaussian-integer
D bit for bit; singular D flagged.

Tolerance per matrix: max |Dinv_gpu - Dinv_oracle| / max |Dinv_oracle| <= TOL * cond_2(D D*)
(the error of this route scales with cond(A) = cond(D)^2)."""
import numpy as np
import pytest
import torch

import oracle
import paper_1111_4144_b200 as hp
from paper_1111_4144_b200 import workloads as wl
from tests import gpu_common as gc

pytestmark = pytest.mark.gpu


def _run(D_dev, layout):
    _, view = wl.to_layout(D_dev, layout)
    Y, info = hp.invert_nonhermitian(view)
    torch.cuda.synchronize()
    return Y.contiguous().cpu().to(torch.complex128).numpy(), info.cpu().numpy()


def _cond_ddh(Dh):
    s = np.linalg.svd(Dh, compute_uv=False)
    return (s[:, 0] / s[:, -1]) ** 2


def _compare(Yg, Yo, infog, infoo, cond, tol):
    assert np.array_equal(infog, infoo), "info mismatch"
    ok = infoo == 0
    if (~ok).any():
        assert np.isnan(Yg[~ok]).all()
    d = np.abs(Yg[ok] - Yo[ok]).reshape(ok.sum(), -1).max(1)
    s = np.abs(Yo[ok]).reshape(ok.sum(), -1).max(1)
    r = d / s / cond[ok]
    assert r.max() <= tol, "err/cond %.3e" % r.max()
    return float(r.max())


def test_cfg7_parity(orc):
    cfg = wl.CONFIGS[7]
    D = wl.generate(cfg, 0, 2 * 4096 + 93, device="cuda")
    Dh = D.cpu().to(torch.complex128).numpy()
    Yo, infoo = oracle.nonherm_batched(Dh)
    for layout in ("aos", "soa"):
        Yg, infog = _run(D, layout)
        _compare(Yg, Yo, infog, infoo, _cond_ddh(Dh), gc.TOL[cfg.dtype])
    assert hp.nonherm_kernel_name(cfg.dtype, cfg.n) == "k_nh_reg<c64>"


@pytest.mark.parametrize("n", list(range(1, 10)) + [16, 33])
@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
def test_all_sizes(orc, n, dtype):
    cfg = wl.Config(94, n, dtype, 0, "chol", "aos", "nonherm", 2.0 * n ** 0.5, 1.0, task="nonherm")
    D = wl.generate(cfg, 0, 150, device="cuda")
    Dh = D.cpu().to(torch.complex128).numpy()
    Yo, infoo = oracle.nonherm_batched(Dh)
    for layout in ("aos", "soa"):
        Yg, infog = _run(D, layout)
        _compare(Yg, Yo, infog, infoo, _cond_ddh(Dh), gc.TOL[dtype])


@pytest.mark.parametrize("n", [4, 8, 12])
@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
def test_exact_gaussian_integer(n, dtype):
    """D = R* P with R unit upper bidiagonal ({+-1, +-i} superdiagonal) and P a signed
    permutation: D D* = R* R exactly, its Cholesky factor is R (unit pivots), and A^-1, D^-1 =
    P^T R^-* are Gaussian integers -- every step is exact, so D^-1 must come back bit for bit."""
    rng = np.random.default_rng(31 + n)
    Ds, Yx = [], []
    units = np.array([1, -1, 1j, -1j])
    for _ in range(50):
        R = np.eye(n, dtype=complex)
        R[np.arange(n - 1), np.arange(1, n)] = units[rng.integers(0, 4, n - 1)]
        P = np.eye(n)[rng.permutation(n)] * rng.choice([-1, 1], n)
        D = R.conj().T @ P
        Yi = np.linalg.inv(D)
        Ds.append(D)
        Yx.append(np.round(Yi.real) + 1j * np.round(Yi.imag))
    D = torch.as_tensor(np.array(Ds)).to(dtype).cuda()
    Yg, info = _run(D, "aos")
    assert (info == 0).all()
    assert np.array_equal(Yg, np.array(Yx))


def test_singular_flagged(orc):
    cfg = wl.CONFIGS[7]
    D = wl.generate(cfg, 0, 64, device="cuda")
    D[5] = 0
    Dh = D.cpu().to(torch.complex128).numpy()
    Yo, infoo = oracle.nonherm_batched(Dh)
    Yg, infog = _run(D, "aos")
    assert infoo[5] > 0
    assert np.array_equal(infog[[5]], infoo[[5]])
    assert np.isnan(Yg[5]).all()


def test_padded_layouts_match(orc):
    cfg = wl.CONFIGS[7]
    D = wl.generate(cfg, 0, 1000, device="cuda")
    Y1, i1 = hp.invert_nonhermitian(D)
    _, Dv = wl.to_layout(D, "soa", ld=1000 + 24)
    Y2, i2 = hp.invert_nonhermitian(Dv)
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2.contiguous()) and torch.equal(i1, i2)


@pytest.mark.parametrize("layout", ["soa", "aos"])
def test_host_pipeline_matches_device(layout):
    """hpdinv_inv_host(method 2) -- D from pinned host memory, chunked -- equals the device call."""
    cfg = wl.CONFIGS[7]
    B = 3000
    D = wl.generate(cfg, 0, B, device="cuda")
    _, Dv = wl.to_layout(D, layout)
    Yd, idv = hp.invert_nonhermitian(Dv)
    torch.cuda.synchronize()
    store, _ = wl.to_layout(D.cpu(), layout)
    store = store.pin_memory()
    Dh = wl.soa_view(store, B, cfg.n) if layout == "soa" else store
    Xh = torch.empty_like(store).pin_memory()
    xh = wl.soa_view(Xh, B, cfg.n) if layout == "soa" else Xh
    xh, ih = hp.invert_host(Dh, "nonherm", xh, chunk=1024)
    torch.cuda.synchronize()
    assert torch.equal(ih, idv.cpu())
    assert torch.equal(xh.contiguous(), Yd.cpu().contiguous())
