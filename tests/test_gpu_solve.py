"""batched linear solve A x = y with the same factorisation
(Cholesky eqs. 5-7, LDL eqs. 12-14): CUDA path vs the fp64 oracle (oracle_solve_batched) on
the same seeded inputs, exact Gaussian-integer systems, info flags, full size sampled.

Tolerance per system b (the north_star's normwise reading R13 applied to x):
  max_i |x_gpu - x_oracle| / max_i |x_oracle| <= TOL * cond_2(A_b).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1111_4144_b200 as hp
from paper_1111_4144_b200 import workloads as wl
from tests import exact
from tests import gpu_common as gc

pytestmark = pytest.mark.gpu


def _run(A_dev, Y_dev, method, layout, vlayout=None):
    _, view = wl.to_layout(A_dev, layout)
    _, yv = wl.vec_layout(Y_dev, vlayout or layout)
    x, info = hp.solve(view, yv, method)
    torch.cuda.synchronize()
    return x.contiguous().cpu().to(torch.complex128).numpy(), info.cpu().numpy()


def _compare(xg, xo, infog, infoo, cond, tol):
    assert np.array_equal(infog, infoo), "info mismatch"
    ok = infoo == 0
    if (~ok).any():
        assert np.isnan(xg[~ok]).all(), "flagged systems must be NaN"
    d = np.abs(xg[ok] - xo[ok]).max(axis=1)
    s = np.abs(xo[ok]).max(axis=1)
    r = d / s / cond[ok]
    assert r.max() <= tol, "err/cond %.3e" % r.max()
    return float(r.max())


def test_cfg6_parity(orc):
    cfg = wl.CONFIGS[6]
    batch = 3 * 4096 + 77                   # several tiles + a ragged tail
    A = wl.generate(cfg, 0, batch, device="cuda")
    Y = wl.generate_rhs(cfg, 0, batch, device="cuda")
    xg, infog = _run(A, Y, cfg.method, cfg.layout)
    Ah = gc.to_host_c128(A)
    xo, infoo = oracle.solve_batched(Ah, Y.cpu().to(torch.complex128).numpy(), cfg.method)
    print("cfg6 worst err/cond = %.3e" % _compare(xg, xo, infog, infoo, gc.cond2(Ah), gc.TOL[cfg.dtype]))
    assert hp.solve_kernel_name(cfg.method, cfg.dtype, cfg.n).startswith("k_solve_reg")


@pytest.mark.parametrize("n", list(range(1, 10)) + [16, 17, 32, 64])
@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
@pytest.mark.parametrize("method", ["chol", "ldl"])
def test_all_sizes(orc, n, dtype, method):
    """Register kernel (n <= 8 / 6) and CTA kernel (above) in both layouts and both dtypes."""
    cfg = wl.Config(98, n, dtype, 0, method, "aos", "bbh", float(n), 0.1, task="solve")
    A = wl.generate(cfg, 0, 261, device="cuda")
    Y = wl.generate_rhs(cfg, 0, 261, device="cuda")
    Ah = gc.to_host_c128(A)
    xo, infoo = oracle.solve_batched(Ah, Y.cpu().to(torch.complex128).numpy(), method)
    for layout, vlayout in (("aos", "aos"), ("soa", "soa"), ("soa", "aos")):
        xg, infog = _run(A, Y, method, layout, vlayout)
        _compare(xg, xo, infog, infoo, gc.cond2(Ah), gc.TOL[dtype])


UNITS = [1, -1, 1j, -1j]


@pytest.mark.parametrize("n", [2, 5, 8, 16, 33])
@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
@pytest.mark.parametrize("method", ["chol", "ldl"])
def test_exact_gaussian_integer_systems(n, dtype, method):
    """A = R*R with R unit upper bidiagonal (superdiagonal in {+-1, +-i}) and an integer x:
    y = A x is exact, every intermediate of eqs. (5)-(7) / (12)-(14) is a small Gaussian
    integer, so the solve must return x bit for bit."""
    rng = np.random.default_rng(100 + n)
    As, ys, xs = [], [], []
    for _ in range(70):
        c = [UNITS[k] for k in rng.integers(0, 4, n - 1)]
        A, _ = exact.bidiag_family(c)
        A = np.array(A)
        x = rng.integers(-3, 4, n) + 1j * rng.integers(-3, 4, n)
        As.append(A)
        xs.append(x)
        ys.append(A @ x)
    A = torch.as_tensor(np.array(As)).to(dtype).cuda()
    Y = torch.as_tensor(np.array(ys)).to(dtype).cuda()
    for layout in ("aos", "soa"):
        xg, info = _run(A, Y, method, layout)
        assert (info == 0).all()
        assert np.array_equal(xg, np.array(xs)), (n, dtype, method, layout)


@pytest.mark.parametrize("n", [3, 8, 20])
@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
@pytest.mark.parametrize("method", ["chol", "ldl"])
def test_info_injection(orc, n, dtype, method):
    """Non-PD systems (clear-margin negative pivots at a chosen index): info bit-exact with
    the oracle, x NaN; the other systems of the batch unaffected."""
    cfg = wl.Config(97, n, dtype, 0, method, "aos", "bbh", float(n), 0.1, task="solve")
    A = wl.generate(cfg, 0, 50, device="cuda")
    Y = wl.generate_rhs(cfg, 0, 50, device="cuda")
    for b, k in ((3, 0), (17, n // 2), (41, n - 1)):
        A[b, k, k] = -5.0 * float(n)
    Ah = gc.to_host_c128(A)
    xo, infoo = oracle.solve_batched(Ah, Y.cpu().to(torch.complex128).numpy(), method)
    assert (infoo[[3, 17, 41]] > 0).all()
    xg, infog = _run(A, Y, method, "aos")
    _compare(xg, xo, infog, infoo, gc.cond2(Ah), gc.TOL[dtype])


def test_bad_args():
    A = torch.zeros(4, 8, 8, dtype=torch.complex64, device="cuda")
    with pytest.raises(ValueError):
        hp.solve(A, torch.zeros(4, 7, dtype=torch.complex64, device="cuda"))
    with pytest.raises(TypeError):
        hp.solve(A, torch.zeros(4, 8, dtype=torch.complex128, device="cuda"))
    x, info = hp.solve(A[:0], torch.zeros(0, 8, dtype=torch.complex64, device="cuda"))
    assert x.shape == (0, 8)


def test_full_size_sampled(orc):
    """cfg6 at its full size in the launch configuration bench.py times: 1500 sampled systems
    vs the oracle one by one, and the residual ||A x - y|| over the whole batch."""
    cfg = wl.CONFIGS[6]
    A = wl.generate(cfg, 0, cfg.batch, device="cuda")
    Y = wl.generate_rhs(cfg, 0, cfg.batch, device="cuda")
    _, view = wl.to_layout(A, cfg.layout)
    _, yv = wl.vec_layout(Y, cfg.layout)
    x, info = hp.solve(view, yv, cfg.method)
    torch.cuda.synchronize()
    assert int((info != 0).sum()) == 0
    rng = np.random.default_rng(6)
    idx = np.unique(np.concatenate([rng.integers(0, cfg.batch, 1500), [0, cfg.batch - 1]]))
    it = torch.as_tensor(idx, device="cuda")
    Ah = gc.to_host_c128(A[it])
    xo, infoo = oracle.solve_batched(Ah, Y[it].cpu().to(torch.complex128).numpy(), cfg.method)
    xs = x[it].cpu().to(torch.complex128).numpy()
    _compare(xs, xo, info[it].cpu().numpy(), infoo, gc.cond2(Ah), gc.TOL[cfg.dtype])
    step = 1 << 16
    for s in range(0, cfg.batch, step):
        Ac = A[s:s + step].to(torch.complex128)
        r = torch.matmul(Ac, x[s:s + step].to(torch.complex128).unsqueeze(-1)).squeeze(-1)
        r -= Y[s:s + step].to(torch.complex128)
        rel = (r.abs().amax(1) / Y[s:s + step].abs().amax(1)).max().item()
        assert rel <= 1e-3, rel


@pytest.mark.parametrize("n", [4, 8, 12])
def test_inplace_padded_and_side_stream(orc, n):
    """Xv aliasing Y with identical strides (header contract), padded interleaved ld for A and
    the vectors, a non-default stream: same results as the plain call."""
    cfg = wl.Config(93, n, torch.complex64, 0, "chol", "soa", "bbh", float(n), 0.1, task="solve")
    B = 777
    A = wl.generate(cfg, 0, B, device="cuda")
    Y = wl.generate_rhs(cfg, 0, B, device="cuda")
    ref, rinfo = hp.solve(A, Y.clone())
    _, Av = wl.to_layout(A, "soa", ld=B + 37)
    _, Yv = wl.vec_layout(Y, "soa", ld=B + 11)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        x, info = hp.solve(Av, Yv, "chol", Xv=Yv, stream=s)
    s.synchronize()
    assert x.data_ptr() == Yv.data_ptr()
    assert torch.equal(x.contiguous(), ref.contiguous()) and torch.equal(info, rinfo)


@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("n", [4, 8, 20])
def test_solve_host_matches_device(n, layout):
    """hpdinv_solve_host (chunked H2D -> kernel -> D2H from pinned host buffers) returns the
    device solve's x and info bit for bit, including a ragged last chunk."""
    cfg = wl.Config(92, n, torch.complex64, 0, "chol", layout, "bbh", float(n), 0.1, task="solve")
    B = 5000
    A = wl.generate(cfg, 0, B, device="cuda")
    Y = wl.generate_rhs(cfg, 0, B, device="cuda")
    A[17, 2, 2] = -50.0                                 # one flagged system
    _, Av = wl.to_layout(A, layout)
    _, Yv = wl.vec_layout(Y, layout)
    xd, idv = hp.solve(Av, Yv, "chol")
    torch.cuda.synchronize()
    As, _ = wl.to_layout(A.cpu(), layout)
    Ys, _ = wl.vec_layout(Y.cpu(), layout)
    As, Ys = As.pin_memory(), Ys.pin_memory()
    if layout == "soa":
        Ah = wl.soa_view(As, B, n)
        Yh = torch.as_strided(Ys, (B, n), (1, B))
    else:
        Ah, Yh = As, Ys
    xh, ih = hp.solve_host(Ah, Yh, "chol", chunk=1536)
    torch.cuda.synchronize()
    assert torch.equal(ih, idv.cpu()) and int(ih[17]) > 0
    assert torch.equal(torch.nan_to_num(xh.contiguous()), torch.nan_to_num(xd.cpu().contiguous()))
