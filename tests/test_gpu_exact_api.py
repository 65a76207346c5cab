"""GPU exactness pins, info flags, API contract, determinism and slicing invariance."""
import ctypes
from math import comb

import numpy as np
import pytest
import torch

import paper_1111_4144_b200 as hp
from paper_1111_4144_b200 import workloads as wl
from tests import exact
from tests import gpu_common as gc

pytestmark = pytest.mark.gpu

UNITS = [1, -1, 1j, -1j]


def _batch_bidiag(n, batch, seed):
    rng = np.random.default_rng(seed)
    As, Xs = [], []
    for _ in range(batch):
        c = [UNITS[k] for k in rng.integers(0, 4, n - 1)]
        A, X = exact.bidiag_family(c)
        As.append(A)
        Xs.append(X)
    return np.array(As), np.array(Xs)


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64])
@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
@pytest.mark.parametrize("method", ["chol", "ldl"])
@pytest.mark.parametrize("layout", ["soa", "aos"])
def test_unit_bidiagonal_exact(n, dtype, method, layout):
    """Gaussian-integer family: the GPU result must equal the exact X bit for bit."""
    As, Xs = _batch_bidiag(n, 67, n)
    A = torch.as_tensor(As).to(dtype).cuda()
    Xg, info, _ = gc.run_gpu(A, method, layout)
    assert (info == 0).all()
    assert np.array_equal(Xg, Xs)


@pytest.mark.parametrize("dtype,nmax", [(torch.complex64, 12), (torch.complex128, 24)])
@pytest.mark.parametrize("method", ["chol", "ldl"])
def test_pascal_exact(dtype, nmax, method):
    for n in range(1, nmax + 1):
        P = np.array(exact.pascal(n), dtype=float)
        u = np.array([1j ** k for k in range(n)])
        u = np.round(u.real) + 1j * np.round(u.imag)
        Pc = (u[:, None] * P) * np.conj(u)[None, :]          # complex Pascal (similarity)
        Xe = (u[:, None] * np.array(exact.pascal_inverse(n), float)) * np.conj(u)[None, :]
        A = torch.as_tensor(np.stack([P + 0j, Pc] * 3)).to(dtype).cuda()
        Xg, info, _ = gc.run_gpu(A, method, "aos")
        assert (info == 0).all()
        want = np.stack([np.array(exact.pascal_inverse(n), float) + 0j, Xe] * 3)
        assert np.array_equal(Xg, want), (n, dtype, method)


@pytest.mark.parametrize("n", [3, 8, 16, 32, 64])
@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
@pytest.mark.parametrize("method", ["chol", "ldl"])
def test_info_injection(orc, n, dtype, method):
    """Clear-margin failures: a_kk := -|a_kk| -> k; zero matrix -> 1; NaN at a_kk -> k;
    NaN in the strict lower triangle -> 0 (never read); Im a_ii poisoned -> ignored."""
    cfg = wl.Config(98, n, dtype, 0, method, "aos", "bbh", float(n), 0.5)
    A = wl.generate(cfg, 0, 64, device="cuda").clone()
    expect = np.zeros(64, np.int32)
    for b in range(0, 40, 5):
        k = (b * 7) % n
        A[b, k, k] = -10.0 * abs(A[b, k, k].item()) - 100.0
        expect[b] = k + 1
    A[41] = 0
    expect[41] = 1
    A[42, n - 1, n - 1] = float("nan")
    expect[42] = n
    if n > 1:
        A[43, n - 1, 0] = float("nan")      # strict lower: not read
        A[44, 0, 0] = complex(A[44, 0, 0].real.item(), 1e30)   # Im a_ii ignored
    A[45, 0, 0] = float("-inf")             # -Inf radicand at pivot 1
    expect[45] = 1
    Ah = gc.to_host_c128(A)
    Xo, infoo = gc.oracle_run(Ah, method)
    for layout in ("aos", "soa"):
        Xg, infog, _ = gc.run_gpu(A, method, layout)
        assert np.array_equal(infog[:46], expect[:46])
        assert np.array_equal(infog, infoo)
        gc.check_mirror(Xg, infog)


def test_batch_zero_and_bad_args():
    L = hp.lib()
    z = ctypes.c_void_p(0)
    assert L.chol_inv_batched_c64(0, 4, z, 16, 1, z, 16, 1, z, z) == 0
    assert L.chol_inv_batched_c64(-1, 4, z, 16, 1, z, 16, 1, z, z) == -1
    assert L.chol_inv_batched_c64(8, 0, z, 16, 1, z, 16, 1, z, z) == -2
    assert L.chol_inv_batched_c64(8, 65, z, 16, 1, z, 16, 1, z, z) == -2
    assert L.chol_inv_batched_c64(8, 4, z, 16, 1, z, 16, 1, z, z) == -3
    A = torch.zeros(8, 4, 4, dtype=torch.complex64, device="cuda")
    X = torch.zeros_like(A)
    info = torch.zeros(8, dtype=torch.int32, device="cuda")
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    assert L.chol_inv_batched_c64(8, 4, p(A), 3, 1, p(X), 16, 1, p(info), z) == -4   # overlap
    assert L.chol_inv_batched_c64(8, 4, p(A), 16, 1, z, 16, 1, p(info), z) == -6
    assert L.chol_inv_batched_c64(8, 4, p(A), 16, 1, p(X), 2, 2, p(info), z) == -7
    assert L.chol_inv_batched_c64(8, 4, p(A), 16, 1, p(X), 16, 1, z, z) == -9
    Ab = ctypes.c_void_p(A.data_ptr() + 4)                                            # misaligned
    assert L.chol_inv_batched_c64(8, 4, Ab, 16, 1, p(X), 16, 1, p(info), z) == -3
    with pytest.raises(TypeError):
        hp.chol_inv_batched_c64(A.to(torch.complex128))
    with pytest.raises(ValueError):
        hp.chol_inv_batched_c64(A.cpu())


@pytest.mark.parametrize("cid", [1, 2, 5])
def test_inplace_padded_stream(orc, cid):
    """X == A in place; padded ld; a non-default stream; no device allocation by the library."""
    cfg = wl.CONFIGS[cid]
    batch = 2000 if cid != 1 else cfg.batch
    A = wl.generate(cfg, 0, batch, device="cuda")
    Ah = gc.to_host_c128(A)
    Xo, infoo = gc.oracle_run(Ah, cfg.method)
    cond = gc.cond2(Ah)
    # padded interleaved layout, out of place, on a side stream
    _, view = wl.to_layout(A, "soa", ld=batch + 37)
    X = wl.empty_like_layout(view)
    info = torch.empty(batch, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    with torch.cuda.stream(s):
        hp.invert(view, cfg.method, X=X, info=info, stream=s)
    s.synchronize()
    assert torch.cuda.memory_allocated() == before
    gc.compare(X.contiguous().cpu().to(torch.complex128).numpy(), Xo, info.cpu().numpy(), infoo,
               cond, gc.TOL[cfg.dtype])
    # in place, both layouts
    for layout in ("soa", "aos"):
        _, v = wl.to_layout(A, layout)
        ref = v.clone() if layout == "aos" else None
        Xi, infoi = hp.invert(v, cfg.method, X=v)
        torch.cuda.synchronize()
        gc.compare(Xi.contiguous().cpu().to(torch.complex128).numpy(), Xo, infoi.cpu().numpy(),
                   infoo, cond, gc.TOL[cfg.dtype])
        del ref


def test_determinism_and_slicing_invariance():
    """Two runs are bitwise equal, and W slices run separately equal the unsliced run: the
    multi-GPU batch slicing cannot change any output bit."""
    for cid in (2, 3, 5):
        cfg = wl.CONFIGS[cid]
        batch = 12345
        A = wl.generate(cfg, 0, batch, device="cuda")
        X1, i1, _ = gc.run_gpu(A, cfg.method, cfg.layout)
        X2, i2, _ = gc.run_gpu(A, cfg.method, cfg.layout)
        assert np.array_equal(X1, X2) and np.array_equal(i1, i2)
        for world in (2, 3, 8):
            parts = []
            for r in range(world):
                s, c = wl.shard(r, world, batch)
                As = wl.generate(cfg, s, c, device="cuda")
                assert torch.equal(As, A[s:s + c])          # chunk-keyed generation
                parts.append(gc.run_gpu(As, cfg.method, cfg.layout)[0])
            assert np.array_equal(np.concatenate(parts), X1)


def test_dmma_schedule_invariance():
    """k_dmma (persistent, one matrix per warp, TMA prefetch of the next matrix during the store
    phase): the output bits do not depend on which warp inverts which matrix or on how many
    matrices a warp chains -- repeated runs, shards of the batch (different grids), in-place
    and padded-stride runs are bitwise equal.  compute-sanitizer is closed on this pool
    (profiles/r02_sanitizer_closed.txt); a race on the shared tiles or the mbarriers would show
    up here as a schedule-dependent result."""
    cfg = wl.CONFIGS[4]
    batch = 3001                                       # > 148 x 6 warps: every warp chains matrices
    A = wl.generate(cfg, 0, batch, device="cuda")
    assert hp.kernel_name("chol", cfg.dtype, batch, cfg.n, (A.stride(0), A.stride(2))) == "k_dmma<c128,chol>"
    X1, i1 = hp.invert(A, "chol")
    X2, i2 = hp.invert(A, "chol")
    torch.cuda.synchronize()
    assert torch.equal(X1, X2) and torch.equal(i1, i2) and int(i1.abs().sum()) == 0
    for world in (2, 7, 40):                           # 40 shards: grids of 13 CTAs, one matrix per warp
        for r in range(world):
            s, c = wl.shard(r, world, batch)
            Xs, _ = hp.invert(A[s:s + c].clone(), "chol")
            assert torch.equal(Xs, X1[s:s + c])
    Ain = A.clone()
    hp.invert(Ain, "chol", X=Ain)                      # in place
    pad = torch.zeros(batch, 64 * 64 + 8, dtype=A.dtype, device="cuda")   # padded matrix stride
    pad[:, :4096] = A.reshape(batch, 4096)
    Ap = torch.as_strided(pad, (batch, 64, 64), (64 * 64 + 8, 64, 1))
    Xp, _ = hp.invert(Ap, "chol")
    torch.cuda.synchronize()
    assert torch.equal(Ain, X1) and torch.equal(Xp.contiguous(), X1)
    # X written by per-lane stores instead of the TMA tensor store (interleaved X)
    Xe = torch.full((64, 64, batch), float("nan"), dtype=A.dtype, device="cuda").permute(2, 0, 1)
    hp.invert(A, "chol", X=Xe)
    torch.cuda.synchronize()
    assert torch.equal(Xe.contiguous(), X1)
    # non-PD matrices in the stream (the NaN store path between TMA-stored neighbours)
    An = A.clone()
    bad = torch.tensor([0, 5, 887, 888, 1500, batch - 1], device="cuda")
    An[bad, 40, 40] = -1.0
    Xn, inf_n = hp.invert(An, "chol")
    torch.cuda.synchronize()
    ok = torch.ones(batch, dtype=torch.bool, device="cuda")
    ok[bad] = False
    assert bool((inf_n[bad] > 0).all()) and int(inf_n[ok].abs().sum()) == 0
    assert bool(torch.isnan(Xn[bad]).all()) and torch.equal(Xn[ok], X1[ok])


def test_kernel_names():
    assert hp.kernel_name("chol", torch.complex64, 1 << 20, 8, (1, 1 << 20)) is not None
    assert hp.kernel_name("chol", torch.complex64, 8, 65) is None


@pytest.mark.parametrize("n", [9, 13, 16])
@pytest.mark.parametrize("method", ["chol", "ldl"])
def test_grp_staged_io_invariance(n, method):
    """k_grp's staged global I/O (bulk copies of whole CTA plane segments through shared memory,
    taken for interleaved A/X with even plane strides and 16-byte aligned bases) and its
    per-lane path (odd plane stride, or an 8-byte aligned X) give bitwise the same X and info,
    full CTAs, a ragged last CTA and NaN-filled flagged matrices included."""
    cfg = wl.Config(97, n, torch.complex64, 0, method, "soa", "bbh", float(n), 0.1)
    batch = 5 * 32 + 19
    A = wl.generate(cfg, 0, batch, device="cuda").clone()
    A[7, n // 2, n // 2] = -1.0                      # flagged inside a full CTA
    A[batch - 3, 0, 0] = -2.0                        # flagged in the ragged CTA
    Xs, is_, _ = gc.run_gpu(A, method, "soa")                    # staged (ld = batch, even)
    Xp, ip, _ = gc.run_gpu(A, method, "soa", ld=batch + 1)       # odd plane stride: per-lane path
    assert np.array_equal(is_, ip) and is_[7] != 0 and is_[batch - 3] == 1
    assert np.array_equal(Xs.view(np.float64), Xp.view(np.float64), equal_nan=True)
    # X base 8-byte aligned only: per-lane stores
    _, view = wl.to_layout(A, "soa")
    store = torch.empty(n * n * batch + 1, dtype=A.dtype, device="cuda")
    X = torch.as_strided(store[1:], view.shape, view.stride())
    X, info = hp.invert(view, method, X=X)
    torch.cuda.synchronize()
    Xm = X.contiguous().cpu().to(torch.complex128).numpy()
    assert np.array_equal(info.cpu().numpy(), is_)
    assert np.array_equal(Xm.view(np.float64), Xs.view(np.float64), equal_nan=True)
