"""Host-side logic of the multi-GPU path, on CPU: chunk-keyed generation, sharding, the
layout helpers, and a world_size-2 gloo run of the bench's slice/timing reduction."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1111_4144_b200 import workloads as wl


def test_shard_covers_batch():
    for batch in (0, 1, 7, 1024, 12345):
        for world in (1, 2, 3, 8):
            parts = [wl.shard(r, world, batch) for r in range(world)]
            assert sum(c for _, c in parts) == batch
            pos = 0
            for s, c in parts:
                assert s == pos
                pos += c


def test_chunk_keyed_generation_is_slice_invariant():
    cfg = wl.CONFIGS[2]
    full = wl.generate(cfg, 0, 3 * wl.CHUNK + 100)
    for s, c in [(0, 10), (wl.CHUNK - 3, 7), (2 * wl.CHUNK + 50, wl.CHUNK + 20)]:
        assert torch.equal(wl.generate(cfg, s, c), full[s:s + c])
    assert not torch.equal(wl.generate(cfg, 0, 10, seed=1), full[:10])


@pytest.mark.parametrize("cid", [1, 2, 3, 5])
def test_generated_matrices_are_hpd_and_hermitian(cid):
    cfg = wl.CONFIGS[cid]
    A = wl.generate(cfg, 0, 64)
    assert torch.equal(A, A.conj().transpose(1, 2))
    assert (torch.diagonal(A, dim1=1, dim2=2).imag == 0).all()
    w = np.linalg.eigvalsh(A.to(torch.complex128).numpy())
    assert (w[:, 0] > 0).all()


def test_spectral_config_conditioning():
    cfg = wl.CONFIGS[4]
    A = wl.generate(cfg, 0, 8)
    w = np.linalg.eigvalsh(A.numpy())
    assert (w[:, 0] >= 1 - 1e-9).all() and (w[:, -1] <= 1e3 * (1 + 1e-9)).all()


def test_layouts_roundtrip():
    cfg = wl.CONFIGS[2]
    A = wl.generate(cfg, 0, 50)
    store, view = wl.to_layout(A, "soa", ld=64)
    assert store.shape == (64, 64) and view.stride() == (1, 8 * 64, 64)
    assert torch.equal(view.contiguous(), A)
    store, view = wl.to_layout(A, "aos")
    assert torch.equal(view, A)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = wl.CONFIGS[2]
    B = 300
    # weak scaling as bench.py: rank r owns [r*B, (r+1)*B) of a global batch of world*B
    A = wl.generate(cfg, rank * B, B)
    t = torch.tensor([float(rank + 1), 10.0 - rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)            # max-over-ranks timing
    gathered = [torch.empty_like(A) for _ in range(world)]
    dist.all_gather(gathered, A)
    if rank == 0:
        q.put((t.tolist(), torch.cat(gathered)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_slices_and_timing():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    t, allA = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert t == [2.0, 10.0]
    assert torch.equal(allA, wl.generate(wl.CONFIGS[2], 0, 600))


def test_rhs_and_fxp_generators_slice_invariant():
    """f1 right-hand sides and f4 fixed-point inputs are chunk-keyed like the matrices: any
    slice equals the same rows of the full draw; the quantised raws stay inside Q(m, f)."""
    cfg6 = wl.CONFIGS[6]
    full = wl.generate_rhs(cfg6, 0, 9000)
    assert torch.equal(full[4000:7000], wl.generate_rhs(cfg6, 4000, 3000))
    cfg8 = wl.CONFIGS[8]
    A, raw = wl.generate_fxp(cfg8, 0, 300)
    A2, raw2 = wl.generate_fxp(cfg8, 100, 50)
    assert torch.equal(A[100:150], A2) and torch.equal(raw[100:150], raw2)
    lim = 2 ** (cfg8.qm + cfg8.qf)
    assert int(raw.max()) <= lim - 1 and int(raw.min()) >= -lim
    assert torch.equal(A, A.conj().transpose(1, 2))
    assert torch.linalg.eigvalsh(A).min() > 0


def test_vector_layouts_roundtrip():
    Y = wl.generate_rhs(wl.CONFIGS[6], 0, 77)
    for layout, ld in (("aos", None), ("soa", None), ("soa", 91)):
        store, view = wl.vec_layout(Y, layout, ld)
        assert torch.equal(view.contiguous(), Y)
        if layout == "soa":
            assert view.stride() == (1, ld or 77)
