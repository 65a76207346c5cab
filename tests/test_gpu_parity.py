"""CUDA path vs the fp64 oracle on the same seeded inputs (BASELINE.json configs 1-5).

Reduced batches span several tiles plus a ragged tail; oracle comparisons are element by
element with the per-matrix tolerance of BASELINE.json's north_star (R13); info
flags must agree bit-exactly.
"""
import numpy as np
import pytest
import torch

from paper_1111_4144_b200 import workloads as wl
from tests import gpu_common as gc

pytestmark = pytest.mark.gpu

# (config id, reduced batch): several tiles of every kernel + a ragged tail
REDUCED = {1: 1024, 2: 3 * 4096 + 77, 3: 2 * 4096 + 131, 4: 301, 5: 4096 + 45}


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_config_parity(orc, cid):
    cfg = wl.CONFIGS[cid]
    A = wl.generate(cfg, 0, REDUCED[cid], device="cuda")
    Xg, infog, _ = gc.run_gpu(A, cfg.method, cfg.layout)
    Ah = gc.to_host_c128(A)
    Xo, infoo = gc.oracle_run(Ah, cfg.method)
    worst = gc.compare(Xg, Xo, infog, infoo, gc.cond2(Ah), gc.TOL[cfg.dtype])
    gc.check_mirror(Xg, infog)
    print("cfg%d worst err/cond = %.3e" % (cid, worst))


@pytest.mark.parametrize("cid", [1, 2, 3, 5])
@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("method", ["chol", "ldl"])
def test_other_layouts_and_methods(orc, cid, layout, method):
    """Every (layout, method) combination on the c64 config ensembles."""
    cfg = wl.CONFIGS[cid]
    A = wl.generate(cfg, 0, 1000 + cid, device="cuda")
    Xg, infog, _ = gc.run_gpu(A, method, layout)
    Ah = gc.to_host_c128(A)
    Xo, infoo = gc.oracle_run(Ah, method)
    gc.compare(Xg, Xo, infog, infoo, gc.cond2(Ah), gc.TOL[cfg.dtype])
    gc.check_mirror(Xg, infog)


@pytest.mark.parametrize("n", list(range(1, 17)) + [17, 23, 31, 32, 33, 48, 63, 64])
@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
@pytest.mark.parametrize("method", ["chol", "ldl"])
def test_all_sizes(orc, n, dtype, method):
    """Every supported size class (register, lane-group and CTA kernels) in both dtypes."""
    cfg = wl.Config(99, n, dtype, 0, method, "aos", "bbh", float(n), 0.1)
    A = wl.generate(cfg, 0, 333, device="cuda")
    for layout in ("aos", "soa"):
        Xg, infog, _ = gc.run_gpu(A, method, layout)
        Ah = gc.to_host_c128(A)
        Xo, infoo = gc.oracle_run(Ah, method)
        gc.compare(Xg, Xo, infog, infoo, gc.cond2(Ah), gc.TOL[dtype])
        gc.check_mirror(Xg, infog)


@pytest.mark.parametrize("cid", [2, 3, 4, 5])
def test_full_size_sampled(orc, cid):
    """BASELINE.json's full sizes in the launch configuration bench.py times: sampled
    matrices vs the oracle one by one, plus properties over the whole batch."""
    cfg = wl.CONFIGS[cid]
    A = wl.generate(cfg, 0, cfg.batch, device="cuda")
    store, view = wl.to_layout(A, cfg.layout)
    del A
    X = wl.empty_like_layout(view)
    import paper_1111_4144_b200 as hp
    X, info = hp.invert(view, cfg.method, X=X)
    torch.cuda.synchronize()
    assert int((info != 0).sum()) == 0
    rng = np.random.default_rng(cid)
    idx = np.unique(np.concatenate([rng.integers(0, cfg.batch, 1500), [0, cfg.batch - 1]]))
    it = torch.as_tensor(idx, device="cuda")
    As = view[it].contiguous()
    Xs = X[it].contiguous().cpu().to(torch.complex128).numpy()
    Ah = gc.to_host_c128(As)
    Xo, infoo = gc.oracle_run(Ah, cfg.method)
    gc.compare(Xs, Xo, info[it].cpu().numpy(), infoo, gc.cond2(Ah), gc.TOL[cfg.dtype])
    gc.check_mirror(Xs, infoo)
    # properties over the whole batch: Hermitian bit-exact, finite, residual ||AX - I||
    step = 1 << 14
    for s in range(0, cfg.batch, step):
        Xc = X[s:s + step].contiguous()
        Ac = view[s:s + step].contiguous()
        assert torch.equal(Xc, Xc.conj().transpose(1, 2)), "mirror"
        assert torch.isfinite(torch.view_as_real(Xc)).all()
        Ac = torch.triu(Ac) + torch.triu(Ac, 1).conj().transpose(1, 2)
        res = torch.matmul(Ac.to(torch.complex128), Xc.to(torch.complex128))
        res -= torch.eye(cfg.n, dtype=torch.complex128, device="cuda")
        r = torch.linalg.matrix_norm(res).max().item()
        assert r <= (1e-2 if cfg.dtype == torch.complex64 else 1e-8), r
