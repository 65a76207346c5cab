"""hpdinv_inv_host (the host-buffer entry point, bench.py's e2e path) for Cholesky and LDL:
bit-exact against the device call with the same layout classes, for interleaved / contiguous
and mixed A / X layouts, odd chunk sizes, a batch that is not a multiple of the chunk, n = 1
contiguous tensors, and the non-Hermitian method with one-matrix chunks (its input and output
regions must not overlap each other or the info)."""
import numpy as np
import pytest
import torch

import paper_1111_4144_b200 as hp
from paper_1111_4144_b200 import workloads as wl

pytestmark = pytest.mark.gpu


def _host_pair(A, a_layout, x_layout):
    """Pinned host A in a_layout and an empty pinned host X in x_layout, plus device copies."""
    batch, n = A.shape[0], A.shape[1]
    sa, va = wl.to_layout(A, a_layout)
    sa = sa.pin_memory()
    va = torch.as_strided(sa, va.shape, va.stride())
    if x_layout == "soa":
        sx = torch.empty(n * n, batch, dtype=A.dtype).pin_memory()
        vx = wl.soa_view(sx, batch, n)
    else:
        sx = torch.empty(batch, n, n, dtype=A.dtype).pin_memory()
        vx = sx
    return va, vx


def _device_ref(va, vx, method):
    # the same strides on the device
    store = torch.empty(va.untyped_storage().nbytes() // va.element_size(), dtype=va.dtype, device="cuda")
    store.copy_(torch.as_strided(va, (store.numel(),), (1,), 0))
    dA = torch.as_strided(store, va.shape, va.stride())
    xs = torch.empty(vx.untyped_storage().nbytes() // vx.element_size(), dtype=vx.dtype, device="cuda")
    dX = torch.as_strided(xs, vx.shape, vx.stride())
    X, info = hp.invert(dA, method, X=dX)
    torch.cuda.synchronize()
    return X.cpu(), info.cpu()


@pytest.mark.parametrize("method,cid", [("chol", 2), ("chol", 3), ("ldl", 5), ("chol", 4)])
@pytest.mark.parametrize("a_layout,x_layout", [("soa", "soa"), ("aos", "aos"), ("soa", "aos"), ("aos", "soa")])
@pytest.mark.parametrize("chunk", [7, 100])
def test_host_matches_device(method, cid, a_layout, x_layout, chunk):
    cfg = wl.CONFIGS[cid]
    batch = 301 if cfg.n <= 16 else 37
    A = wl.generate(cfg, 0, batch)
    va, vx = _host_pair(A, a_layout, x_layout)
    Xr, ir = _device_ref(va, vx, method)
    Xh, ih = hp.invert_host(va, method, vx, chunk=chunk)
    torch.cuda.synchronize()
    assert torch.equal(ih, ir)
    assert torch.equal(Xh.contiguous(), Xr.contiguous())       # bit for bit, NaN-free inputs
    assert (ih == 0).all()


@pytest.mark.parametrize("method", ["chol", "ldl"])
@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
def test_host_n1_contiguous(method, dtype):
    """n = 1 contiguous (B, 1, 1) tensors (strides (1, 1, 1)): x = 1 / Re a_11 (reading R20)."""
    B = 513
    a = (torch.rand(B, dtype=torch.float64) + 0.5).to(dtype).reshape(B, 1, 1).pin_memory()
    a[7, 0, 0] = -1.0
    X, info = hp.invert_host(a, method, chunk=100)
    torch.cuda.synchronize()
    Xd, infod = hp.invert(a.cuda(), method)
    assert torch.equal(info, infod.cpu())
    assert int(info[7]) == 1 and (info[np.arange(B) != 7] == 0).all()
    assert torch.equal(X[info == 0], Xd.cpu()[infod.cpu() == 0])
    assert torch.isnan(X[7]).all()


@pytest.mark.parametrize("batch,chunk", [(1, 1), (1, 0), (3, 1), (5, 2)])
def test_host_nonherm_small_chunks(batch, chunk):
    """Method 2 (out of place): one-matrix chunks keep D^-1 and info apart."""
    cfg = wl.Config(95, 8, torch.complex64, 0, "chol", "aos", "nonherm", 2.0 * 8 ** 0.5, 1.0, task="nonherm")
    D = wl.generate(cfg, 0, batch)
    Dh = D.pin_memory()
    Yd, idv = hp.invert_nonhermitian(D.cuda())
    Yh, ih = hp.invert_host(Dh, "nonherm", chunk=chunk)
    torch.cuda.synchronize()
    assert torch.equal(ih, idv.cpu())
    assert torch.equal(Yh, Yd.cpu())


def test_host_repeated_calls_reuse_pipeline():
    """The copy streams and events are created once per device and reused: many small calls
    on two user streams stay correct."""
    cfg = wl.CONFIGS[2]
    A = wl.generate(cfg, 0, 64).pin_memory()
    Xr, ir = hp.invert(A.cuda(), "chol")
    Xr = Xr.cpu()
    s2 = torch.cuda.Stream()
    outs = []
    for k in range(40):
        st = s2 if k % 2 else torch.cuda.current_stream()
        outs.append(hp.invert_host(A, "chol", chunk=16, stream=st))
    torch.cuda.synchronize()
    for X, info in outs:
        assert torch.equal(X, Xr) and (info == 0).all()
