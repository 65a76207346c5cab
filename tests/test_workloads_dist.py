"""Host-side logic of the multi-GPU path, on CPU: chunk-keyed generation, sharding, the
layout helpers, and a world_size-2 gloo run of the bench's slice/timing reduction."""
import os
import socket
import time

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


class _CpuBackend:
    """Stand-in for bench.CudaBackend on a CPU-only box: the same prepare/step/timer interface,
    with the fp64 oracle as the step (test infrastructure).  Rank r sleeps r+1 ms per step so
    the max-over-ranks reduction is visible in the result."""

    def __init__(self, rank):
        self.rank = rank
        self.device = torch.device("cpu")
        self.slices = []

    def sync(self):
        pass

    def event(self):
        return time.perf_counter()

    @staticmethod
    def elapsed_ms(a, b):
        return (b - a) * 1e3

    def sampler(self):
        import bench
        return bench.NullSampler()

    def prepare(self, cfg, start, count, args):
        import oracle
        A = wl.generate(cfg, start, count, seed=args.seed)
        Ah = A.to(torch.complex128).numpy()
        st = {"cfg": cfg, "count": count, "kernel": "oracle-cpu", "view": A}
        self.slices.append((cfg.cid, start, count))

        def step():
            X, info = oracle.inv_batched(Ah, cfg.method, nthreads=1)
            st["X"], st["info"] = X, info
            time.sleep(1e-3 * (self.rank + 1))
        st["step"] = step
        return st

    def maybe_graph(self, st, per_step_s, mode):
        return st["step"], "cpu stand-in"

    def nonzero_info(self, st):
        return int((st["info"] != 0).sum())

    def release(self):
        pass


SMALL = {2: 300, 3: 37, 4: 6, 5: 11}


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(2)                           # two ranks share the host's cores
    import dataclasses
    import bench
    for cid, b in SMALL.items():                       # BASELINE shapes, small batches
        wl.CONFIGS[cid] = dataclasses.replace(wl.CONFIGS[cid], batch=b)
    args = bench.parse(["--gpus", str(world), "--steps", "3", "--warmup", "3"])
    be = _CpuBackend(rank)
    heads = {}

    def extras(cfg, st, head):                          # keep the headline's slice result
        heads["X"], heads["info"] = torch.from_numpy(st["X"]), torch.from_numpy(st["info"])
        return {}
    out = bench.run_rank(args, rank, world, bench.Dist(world, torch.device("cpu")), be, extras)
    n = wl.CONFIGS[2].n
    counts = torch.tensor([heads["X"].shape[0]])
    allc = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(allc, counts)
    mx = int(max(c.item() for c in allc))
    pad = torch.zeros(mx, n, n, dtype=torch.complex128)
    pad[:heads["X"].shape[0]] = heads["X"]
    gathered = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(gathered, pad)
    if rank == 0:
        X = torch.cat([g[:int(c.item())] for g, c in zip(gathered, allc)])
        q.put((out, X, be.slices))
    else:
        q.put(("slices", rank, be.slices))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_runs_the_bench_rank_function():
    """bench.run_rank -- the rank function of the GPU run -- under a world-2 gloo group: strong
    scaling shards each fixed global batch into contiguous slices generated on each rank, the
    reported timings are the max over ranks, value = global batch / that time, n_gpus = 2, and
    the gathered headline result equals a one-rank run of the whole batch."""
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    out, X, slices0 = next(g for g in got if not isinstance(g[0], str))
    slices1 = next(g for g in got if isinstance(g[0], str))[2]
    assert out["n_gpus"] == 2 and out["scaling"] == "strong"
    assert out["config"]["global_batch"] == SMALL[2]
    assert abs(out["value"] - SMALL[2] / (out["ms_per_step"] / 1e3)) < 1e-6 * out["value"]
    assert out["ms_per_step"] >= 2.0                  # rank 1 sleeps 2 ms per step: the max is taken
    assert set(out["per_config"]) == {"cfg3", "cfg4", "cfg5"}
    for cid in (3, 4, 5):
        r = out["per_config"]["cfg%d" % cid]
        assert r["n_gpus"] == 2 and r["global_batch"] == SMALL[cid] and r["ms_per_step"] >= 2.0
        assert abs(r["value"] - SMALL[cid] / (r["ms_per_step"] / 1e3)) < 1e-6 * r["value"]
    # the two ranks' slices tile every global batch, in order
    for cid in (2, 3, 4, 5):
        s0 = [(s, c) for k, s, c in slices0 if k == cid][0]
        s1 = [(s, c) for k, s, c in slices1 if k == cid][0]
        assert s0[0] == 0 and s0[0] + s0[1] == s1[0] and s1[0] + s1[1] == SMALL[cid]
    full = wl.generate(wl.CONFIGS[2], 0, SMALL[2]).to(torch.complex128).numpy()
    Xo, _ = oracle.inv_batched(full, "chol", nthreads=1)
    assert np.array_equal(X.numpy(), Xo)


def test_bench_launcher_spawns_and_checks_world(monkeypatch):
    """--gpus N without a torchrun environment re-launches under torch.distributed.run with N
    ranks on 127.0.0.1; inside torchrun a WORLD_SIZE that disagrees with --gpus is an error."""
    import bench
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    assert bench.main(["--gpus", "4", "--steps", "2"]) == 0
    cmd = calls[0]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert cmd[cmd.index("--nproc-per-node") + 1] == "4"
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "0")
    assert bench.main(["--gpus", "4"]) == 2


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
