"""the paper's EXISTING inversion methods on the GPU (equation solving,
eq. 15; triangular matrix operations, eqs. 16-19) vs the fp64 oracle's implementations of the
same methods (oracle_eqsolve_inv / oracle_trimat_inv), on the same seeded inputs; exact
Gaussian-integer family bit for bit; info flags."""
import numpy as np
import pytest
import torch

import oracle
import paper_1111_4144_b200 as hp
from paper_1111_4144_b200 import workloads as wl
from tests import gpu_common as gc
from tests.test_gpu_exact_api import _batch_bidiag

pytestmark = pytest.mark.gpu


def _run(A_dev, method, layout):
    _, view = wl.to_layout(A_dev, layout)
    X, info = hp.invert_method(view, method)
    torch.cuda.synchronize()
    return X.contiguous().cpu().to(torch.complex128).numpy(), info.cpu().numpy()


@pytest.mark.parametrize("n", list(range(1, 10)) + [16, 33])
@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
@pytest.mark.parametrize("method", ["eqsolve", "trimat"])
def test_parity(orc, n, dtype, method):
    cfg = wl.Config(96, n, dtype, 0, "chol", "aos", "bbh", float(n), 0.1)
    A = wl.generate(cfg, 0, 200 + n, device="cuda")
    Ah = gc.to_host_c128(A)
    Xo, infoo = oracle.inv_batched(Ah, method)
    for layout in ("aos", "soa"):
        Xg, infog = _run(A, method, layout)
        gc.compare(Xg, Xo, infog, infoo, gc.cond2(Ah), gc.TOL[dtype])
        gc.check_mirror(Xg, infog)


def test_cfg2_kernel_and_parity(orc):
    cfg = wl.CONFIGS[2]
    A = wl.generate(cfg, 0, 3 * 4096 + 77, device="cuda")
    Ah = gc.to_host_c128(A)
    for method in ("eqsolve", "trimat"):
        assert hp.method_kernel_name(method, cfg.dtype, cfg.n).startswith("k_base_reg")
        Xg, infog = _run(A, method, "soa")
        Xo, infoo = oracle.inv_batched(Ah, method)
        gc.compare(Xg, Xo, infog, infoo, gc.cond2(Ah), gc.TOL[cfg.dtype])


@pytest.mark.parametrize("n", [4, 8, 12])
@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
@pytest.mark.parametrize("method", ["eqsolve", "trimat"])
def test_exact_family(n, dtype, method):
    As, Xs = _batch_bidiag(n, 40, 7 * n)
    A = torch.as_tensor(As).to(dtype).cuda()
    Xg, info = _run(A, method, "aos")
    assert (info == 0).all()
    assert np.array_equal(Xg, Xs)


@pytest.mark.parametrize("n", [3, 8, 20])
@pytest.mark.parametrize("method", ["eqsolve", "trimat"])
def test_info(orc, n, method):
    cfg = wl.Config(95, n, torch.complex64, 0, "chol", "aos", "bbh", float(n), 0.1)
    A = wl.generate(cfg, 0, 40, device="cuda")
    for b, k in ((2, 0), (21, n - 1)):
        A[b, k, k] = -5.0 * n
    Ah = gc.to_host_c128(A)
    Xo, infoo = oracle.inv_batched(Ah, method)
    Xg, infog = _run(A, method, "aos")
    gc.compare(Xg, Xo, infog, infoo, gc.cond2(Ah), gc.TOL[torch.complex64])
    gc.check_mirror(Xg, infog)


def test_proposed_through_method_entry(orc):
    """methods 0 / 1 of hpdinv_inv_batched_method are exactly the proposed entry points."""
    cfg = wl.CONFIGS[3]
    A = wl.generate(cfg, 0, 999, device="cuda")
    _, view = wl.to_layout(A, "soa")
    for m in ("chol", "ldl"):
        X1, i1 = hp.invert_method(view, m)
        X2, i2 = hp.invert(view, m)
        torch.cuda.synchronize()
        assert torch.equal(X1, X2) and torch.equal(i1, i2)
