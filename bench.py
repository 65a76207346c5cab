#!/usr/bin/env python
"""bench.py -- throughput of the batched HPD inversion hot path (BASELINE.json metric).

One step = one pass of the whole hot path (load upper(A) -> Cholesky/LDL -> proposed
inversion -> mirror -> store) over one batch of synthetic matrices, i.e.
one call of the C ABI entry point.  Default workload: BASELINE.json configs[1] (cfg2: 2^20
complex64 8x8 HPD matrices, interleaved layout); the same line carries `per_config` entries
for the other metric sizes (cfg3 N=16, cfg4 N=64, cfg5 N=32 LDL), each timed the same way.
`--config k` makes another workload the headline.

Multi-GPU: `--gpus N` without a torchrun environment re-launches this script
under `torch.distributed.run` with N ranks (one per GPU, NCCL, 127.0.0.1).  Default scaling
is STRONG: the fixed BASELINE global batch B is sharded, rank r owning the contiguous slice
`workloads.shard(r, W, B)` and generating it on its own device from the chunk-keyed seeds;
`--scaling weak` gives every rank a full B instead.  No collective touches the data path:
NCCL carries only the start barrier and the max-over-ranks reduction of the timings.
value = global matrices / max_r (rank r's device time per step).

`--impl reference` times the fp64 CPU oracle (the reference arm of this tier) on bounded
samples of the same workload, on rank 0 only.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1111_4144_b200 import workloads as wl  # noqa: E402

METRIC = "HPD matrices inverted/sec (N=8,16,64) and % of HBM/FP roofline, 1-8 B200"
UNIT = "matrices/s"
METRIC_SOLVE = "HPD linear systems solved/sec (SURVEY 8(f) f1: A x = y, eqs. 5-7 / 12-14), 1 B200"
UNIT_SOLVE = "systems/s"
L2_BYTES = 126 * 2**20
SMS = 148
DEFAULT_PER_CONFIG = {2: "3,4,5"}      # the headline cfg2 line also times the other metric sizes


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, default=2, choices=sorted(wl.CONFIGS))
    p.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                   help="strong: shard the fixed global batch over the ranks (default); weak: a full batch per rank")
    p.add_argument("--per-config", default=None,
                   help="comma list of extra configs timed into `per_config` ('' = none; default 3,4,5 for cfg2)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-library", action="store_true", help="skip the vendor-library comparison")
    p.add_argument("--batch", type=int, default=None,
                   help="override the headline config's global batch (e.g. an L2-resident study; not a BASELINE line)")
    p.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                   help="replay each step from a CUDA graph (auto: for launch-bound per-rank batches)")
    p.add_argument("--inv-method", choices=["proposed", "eqsolve", "trimat"], default="proposed",
                   help="SURVEY 8(f) f3: time one of the paper's existing methods on the GPU instead")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    return p.parse_args(argv)


# ----------------------------------------------------------------------------- helpers
def algorithmic_bytes(cfg: wl.Config) -> int:
    """Per matrix: read the upper triangle, write all n^2 entries of X and one int32 info
    (solve: read the upper triangle and y, write x and info)."""
    n, e = cfg.n, cfg.elem_bytes
    if cfg.task == "solve":
        return e * (n * (n + 1) // 2 + 2 * n) + 4
    if cfg.task == "nonherm":         # read all of D, write D^-1
        return e * 2 * n * n + 4
    return e * (n * (n + 1) // 2 + n * n) + 4


def cmul_per_matrix(n: int, task: str = "inv") -> int:
    if task == "solve":               # factor (n^3-n)/6 + two substitutions n(n-1)/2 each
        return (n ** 3 - n) // 6 + n * (n - 1)
    if task == "nonherm":             # D D* (upper) + Cholesky + proposed + D* X
        return n * n * (n + 1) // 2 + (n ** 3 - n) // 2 + n ** 3
    return (n ** 3 - n) // 2          # Table 1 proposed total, exact


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        mp = json.load(open(path))
        return {"hbm_gbs": float(mp["hbm_gbs"]), "sm_max_mhz": float(mp.get("sm_max_mhz", 1965.0)),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


def fp_peak_tflops(dtype: torch.dtype, mhz: float) -> float:
    """FP32 / FP64 FMA peak from unit counts: 148 SMs x {128, 64} FMA/clk x 2.
    (FP64: the DMMA tensor path measured 37.05 TF/s, `profiles/r02_mma_peaks.txt`, on the same
    FP64 datapath as DFMA -- the derived 37.2 is the larger, so it is the denominator.)"""
    lanes = 128 if dtype == torch.complex64 else 64
    return SMS * lanes * 2 * mhz * 1e6 / 1e12


class ClockSampler:
    """Samples SM clock and clock-event reasons via NVML while the timed region runs."""
    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x100: "display_clock_setting"}

    def __init__(self, cuda_device: int, period_s: float = 0.005):
        self.samples = []
        self.period = period_s
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            pr = torch.cuda.get_device_properties(cuda_device)
            try:
                bus = "%08X:%02X:%02X.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(cuda_device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - depends on the box
            self.err = repr(e)
            self.max_mhz = None

    def _sample(self):
        nv = self.nv
        try:
            mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
            try:
                reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                reasons = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            self.samples.append((mhz, int(reasons)))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self.ok:
            self._sample()
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0,
                    "note": getattr(self, "err", "no samples")}
        mhz = [s[0] for s in self.samples]
        mask = 0
        for s in self.samples:
            mask |= s[1]
        reasons = [v for k, v in self.NAMES.items() if mask & k and k != 0x1]
        return {"sm_mhz": float(statistics.median(mhz)), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


class NullSampler:
    def start(self):
        pass

    def stop(self):
        pass

    def summary(self):
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "note": "no GPU"}


def load_traffic(cfg: wl.Config, kernel: str, batch: int):
    """Per-launch DRAM bytes of this kernel from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        t = json.load(open(path))
        rec = t.get("cfg%d" % cfg.cid)
        if rec and rec.get("kernel") == kernel and rec.get("batch") == batch:
            return float(rec["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


# ------------------------------------------------------------- multi-rank plumbing
class Dist:
    """Barrier and max/min reductions over the ranks (NCCL on the GPU box, gloo in the CPU
    test); a no-op for one rank.  Nothing here touches the data path."""

    def __init__(self, world: int, device):
        self.world = world
        self.device = device

    def barrier(self):
        if self.world > 1:
            if self.device.type == "cuda":
                torch.distributed.barrier(device_ids=[self.device.index])
            else:
                torch.distributed.barrier()

    def _reduce(self, vals, op):
        t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=self.device)
        if self.world > 1:
            torch.distributed.all_reduce(t, op=op)
        return t.tolist()

    def max(self, vals):
        return self._reduce(vals, torch.distributed.ReduceOp.MAX if self.world > 1 else None)

    def min(self, vals):
        return self._reduce(vals, torch.distributed.ReduceOp.MIN if self.world > 1 else None)


def shard_plan(cfg: wl.Config, rank: int, world: int, scaling: str, batch=None):
    """(start, count, global_batch) of this rank.  strong: the fixed global batch B is split
    into contiguous slices ([r B/W, (r+1) B/W)); weak: rank r owns the r-th
    full batch of a global batch of W x B."""
    B = int(batch) if batch else cfg.batch
    if scaling == "weak":
        return rank * B, B, world * B
    start, count = wl.shard(rank, world, B)
    return start, count, B


class CudaBackend:
    """The product path: inputs generated on this rank's GPU, one C-ABI call per step, CUDA
    events on the launching stream."""

    def __init__(self, device):
        import paper_1111_4144_b200 as hp
        self.hp = hp
        self.device = device

    def sync(self):
        torch.cuda.synchronize(self.device)

    def event(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream(self.device))
        return e

    @staticmethod
    def elapsed_ms(a, b):
        return a.elapsed_time(b)

    def sampler(self):
        return ClockSampler(self.device.index)

    def prepare(self, cfg: wl.Config, start: int, count: int, args):
        hp = self.hp
        dev = self.device
        st = {"cfg": cfg, "count": count}
        A = wl.generate(cfg, start, count, device=dev, seed=args.seed)
        store, view = wl.to_layout(A, cfg.layout)
        del A
        st.update(store=store, view=view)
        info = torch.empty(count, dtype=torch.int32, device=dev)
        st["info"] = info
        if cfg.task == "solve":
            Y = wl.generate_rhs(cfg, start, count, device=dev, seed=args.seed)
            ystore, yview = wl.vec_layout(Y, cfg.layout)
            del Y
            Xv = torch.empty_strided(yview.shape, yview.stride(), dtype=cfg.dtype, device=dev)
            st.update(ystore=ystore, yview=yview, X=Xv, kernel=hp.solve_kernel_name(cfg.method, cfg.dtype, cfg.n))
            st["step"] = lambda: hp.solve(view, yview, cfg.method, Xv=Xv, info=info)
        elif cfg.task == "nonherm":
            X = wl.empty_like_layout(view)
            st.update(X=X, kernel=hp.nonherm_kernel_name(cfg.dtype, cfg.n))
            st["step"] = lambda: hp.invert_nonhermitian(view, Dinv=X, info=info)
        elif args.inv_method != "proposed":
            X = wl.empty_like_layout(view)
            st.update(X=X, kernel=hp.method_kernel_name(args.inv_method, cfg.dtype, cfg.n))
            st["step"] = lambda: hp.invert_method(view, args.inv_method, X=X, info=info)
        else:
            X = wl.empty_like_layout(view)
            st.update(X=X, kernel=hp.kernel_name(cfg.method, cfg.dtype, count, cfg.n,
                                                 (view.stride(0), view.stride(2)), (X.stride(0), X.stride(2))))
            st["step"] = lambda: hp.invert(view, cfg.method, X=X, info=info)
        return st

    def maybe_graph(self, st, per_step_s: float, mode: str):
        """Launch-bound per-rank batches (cfg1, or a strong-scaled slice whose kernel is a few
        tens of µs) replay the step from CUDA graphs so the host-side Python/ctypes overhead does
        not pose as kernel time: one graph holds G consecutive steps (G kernel nodes, G * the
        kernel time >= ~100 µs) and one graph a single step, so exactly `steps` launches are
        timed.  Returns (multi_fn, G, single_fn) or a plain per-step callable."""
        use = mode == "on" or (mode == "auto" and per_step_s < 60e-6)
        if not use:
            return st["step"], "direct C-ABI call per step"
        G = max(1, min(64, int(100e-6 / max(per_step_s, 1e-6))))
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1):
            st["step"]()
        gG = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gG):
            for _ in range(G):
                st["step"]()
        g1.replay()
        gG.replay()
        self.sync()
        st["graphs"] = (g1, gG)
        return (gG.replay, G, g1.replay), ("CUDA graphs of the C-ABI call (%d steps = %d kernel nodes per "
                                           "replay, and a one-step graph for the remainder)" % (G, G))

    def nonzero_info(self, st):
        return int((st["info"] != 0).sum().item())

    def release(self):
        torch.cuda.empty_cache()


def timed_loop(step, steps: int, warmup: int, backend, dist: Dist):
    """W untimed warm-up steps, then exactly `steps` timed steps between a barrier +
    synchronize on both sides.  `step` is a per-step callable or (multi_fn, G, single_fn): a
    replay of G steps and of one step (launch-bound batches, see CudaBackend.maybe_graph).
    Returns (ms_per_step, kernel_ms, wall_span_ms) reduced over the ranks: the max of the
    per-rank device times (kernel_ms = event time around the launches / steps); the wall span
    is the host-clock interval from the earliest rank's start to the latest rank's end (ranks
    share one host clock)."""
    if isinstance(step, tuple):
        multi, G, single = step
        plan = [(multi, G)] * (steps // G) + [(single, 1)] * (steps % G)
        warm = [(multi, G)] * (warmup // G) + [(single, 1)] * (warmup % G)
    else:
        plan = [(step, 1)] * steps
        warm = [(step, 1)] * warmup
    for fn, _ in warm:
        fn()
    backend.sync()
    dist.barrier()
    backend.sync()
    t_host0 = time.time()
    t0 = backend.event()
    evs = []
    for fn, _ in plan:
        a = backend.event()
        fn()
        evs.append((a, backend.event()))
    t1 = backend.event()
    backend.sync()
    t_host1 = time.time()
    dist.barrier()
    elapsed = backend.elapsed_ms(t0, t1)
    kern = sum(backend.elapsed_ms(a, b) for a, b in evs) / steps
    elapsed, kern, t_end = dist.max([elapsed, kern, t_host1])
    (t_start,) = dist.min([t_host0])
    return elapsed / steps, kern, (t_end - t_start) * 1e3


def roofline(cfg: wl.Config, count: int, kern_ms: float, kernel: str):
    """Roofline of the (single) kernel of the step on this rank's slice: algorithmic bytes (or
    the paper's multiply count for the FP-bound sizes) per launch / the kernel's event time."""
    pk = peaks()
    bytes_launch = algorithmic_bytes(cfg) * count
    mem_s = bytes_launch / (pk["hbm_gbs"] * 1e9)
    fp_tf = fp_peak_tflops(cfg.dtype, pk["sm_max_mhz"])
    flops_launch = 8.0 * cmul_per_matrix(cfg.n, cfg.task) * count
    fp_s = flops_launch / (fp_tf * 1e12)
    if fp_s > mem_s:
        achieved = flops_launch / (kern_ms / 1e3) / 1e12
        tc = kernel.startswith("k_dmma")
        roof = {"bound": "tensor" if tc else "alu", "achieved": achieved, "peak": fp_tf, "unit": "TFLOP/s",
                "frac": achieved / fp_tf,
                "peak_source": "derived FP%d peak: 148 SMs x %d FMA/clk x 2 x %.0f MHz%s"
                % (32 if cfg.dtype == torch.complex64 else 64, 128 if cfg.dtype == torch.complex64 else 64,
                   pk["sm_max_mhz"], " (FP64 DMMA tensor path; measured DMMA peak 37.05 TF/s, "
                   "profiles/r02_mma_peaks.txt)" if tc else "")}
    else:
        achieved = bytes_launch / (kern_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "peak_source": pk["source"]}
    roof["traffic"] = load_traffic(cfg, kernel, count)
    roof["algorithmic_bytes_per_launch"] = bytes_launch
    roof["flops_per_launch"] = flops_launch
    roof["kernel"] = kernel
    roof["kernel_ms"] = kern_ms
    # BASELINE.json's own formula: max(16 N^2 batch / HBM, multiply count / FP peak)
    bj_bytes = 2 * cfg.elem_bytes * cfg.n ** 2 * count
    bj_t = max(bj_bytes / (pk["hbm_gbs"] * 1e9), fp_s)
    return roof, {"time_s": bj_t, "frac": bj_t / (kern_ms / 1e3), "bytes": bj_bytes,
                  "note": "BASELINE.json north_star formula"}


def config_dict(cfg: wl.Config, world: int, scaling: str, batch=None):
    """The workload description shared by both arms (so the driver sees the same config)."""
    B = int(batch) if batch else cfg.batch
    global_batch = B * world if scaling == "weak" else B
    bj_bytes = 2 * cfg.elem_bytes * cfg.n ** 2 * global_batch
    return {"workload": "cfg%d: %s" % (cfg.cid, cfg.desc), "n": cfg.n, "global_batch": global_batch,
            "elem": "complex64" if cfg.dtype == torch.complex64 else "complex128",
            "method": cfg.method, "layout": cfg.layout,
            "parallelism": "batch sharded over %d rank(s) (%s scaling), no collective" % (world, scaling),
            "l2": ("inputs larger than L2 (%.0f MB > 126 MB); no flush" % (bj_bytes / 1e6)
                   if bj_bytes > L2_BYTES else "working set fits L2")}


def run_config(args, cfg: wl.Config, rank: int, world: int, dist: Dist, backend, steps=None, batch=None):
    """One workload on this rank: generate the rank's slice, time the step, reduce over the
    ranks.  Returns (summary dict, state) -- the state keeps the buffers for e2e and checks."""
    start, count, global_batch = shard_plan(cfg, rank, world, args.scaling, batch)
    st = backend.prepare(cfg, start, count, args)
    per_step_guess = max(algorithmic_bytes(cfg) * count / 6.0e12,
                         8.0 * cmul_per_matrix(cfg.n, cfg.task) * count / 3.0e13, 2e-6)
    if steps is None:
        steps = max(20, min(2000, int(0.5 / per_step_guess)))
    warmup = max(3, args.warmup)
    step, launch = backend.maybe_graph(st, per_step_guess, args.graph)
    sampler = backend.sampler()
    # the warm-up and the timed steps both live inside timed_loop; the sampler runs over it
    sampler.start()
    ms_per_step, kern_ms, wall_ms = timed_loop(step, steps, warmup, backend, dist)
    sampler.stop()
    bad = backend.nonzero_info(st)
    (bad,) = dist.max([bad])
    roof, bj = roofline(cfg, count, kern_ms, st["kernel"])
    out = {
        "value": global_batch / (ms_per_step / 1e3), "unit": UNIT_SOLVE if cfg.task == "solve" else UNIT,
        "ms_per_step": ms_per_step, "kernel_ms": kern_ms, "wall_span_ms": wall_ms, "steps": steps,
        "warmup": warmup, "n_gpus": world, "global_batch": global_batch, "batch_per_rank": count,
        "rank_slice": [start, start + count], "launch": launch, "roofline": roof, "roofline_baseline_formula": bj,
        "clocks": sampler.summary(), "gpu_launches": steps, "info_nonzero": int(bad),
    }
    return out, st


def e2e_measure(args, cfg: wl.Config, st, world: int, dist: Dist, dev, steps: int):
    """The same metric end to end through the host-buffer C entry points (pinned host A [, y]
    -> H2D -> kernel -> D2H of X and info), timed with CUDA events; the result read back must
    match the device-resident run bit for bit."""
    hp = CudaBackend(dev).hp
    B = st["count"]
    store = st["store"]
    stream = torch.cuda.current_stream(dev)
    e2e_steps = max(3, min(steps, 10))
    chunk = max(4096, B // 8)          # 8 chunks: measured best of 4 / 8 / 16 / 32 at cfg2
    if cfg.task == "solve":
        A_host = store.cpu().pin_memory()
        Y_host = st["ystore"].cpu().pin_memory()
        if cfg.layout == "soa":
            vh = wl.soa_view(A_host, B, cfg.n)
            yh = torch.as_strided(Y_host, (B, cfg.n), (1, Y_host.shape[1]))
            h2d = cfg.elem_bytes * (cfg.n * (cfg.n + 1) // 2 + cfg.n) * B
        else:
            vh, yh = A_host, Y_host
            h2d = cfg.elem_bytes * (cfg.n * cfg.n + cfg.n) * B
        X_host = torch.empty_like(Y_host).pin_memory()
        xh = torch.as_strided(X_host, yh.shape, yh.stride())
        info_h = torch.empty(B, dtype=torch.int32).pin_memory()
        ws = torch.empty(hp.solve_host_workspace_bytes(cfg.dtype, cfg.n, chunk), dtype=torch.uint8, device=dev)

        def call():
            hp.solve_host(vh, yh, cfg.method, xh, info_h, ws, chunk)
        d2h = cfg.elem_bytes * cfg.n * B + 4 * B
        unit, api = UNIT_SOLVE, "hpdinv_solve_host (pinned host buffers)"
    else:
        nh = cfg.task == "nonherm"
        A_host = store.cpu().pin_memory()
        X_host = torch.empty_like(A_host).pin_memory()
        if cfg.layout == "soa":
            vh = wl.soa_view(A_host, B, cfg.n)
            xh = wl.soa_view(X_host, B, cfg.n)
            h2d = cfg.elem_bytes * (cfg.n * cfg.n if nh else cfg.n * (cfg.n + 1) // 2) * B
        else:
            vh, xh = A_host, X_host
            h2d = cfg.elem_bytes * cfg.n * cfg.n * B
        info_h = torch.empty(B, dtype=torch.int32).pin_memory()
        ws = torch.empty(hp.host_workspace_bytes(cfg.dtype, cfg.n, chunk), dtype=torch.uint8, device=dev)
        hmethod = "nonherm" if nh else cfg.method

        def call():
            hp.invert_host(vh, hmethod, xh, info_h, ws, chunk)
        d2h = cfg.elem_bytes * cfg.n * cfg.n * B + 4 * B
        unit, api = UNIT, "hpdinv_inv_host (pinned host buffers)"
    for _ in range(2):
        call()
    torch.cuda.synchronize(dev)
    dist.barrier()
    torch.cuda.synchronize(dev)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(e2e_steps):
        call()
    b.record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    (ms,) = dist.max([a.elapsed_time(b) / e2e_steps])
    same = torch.equal(xh.contiguous(), st["X"].cpu().contiguous()) and torch.equal(info_h, st["info"].cpu())
    global_batch = B * world if args.scaling == "weak" else cfg.batch
    return {"value": global_batch / (ms / 1e3), "unit": unit, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": ms, "chunk": chunk,
            "matches_device_run": bool(same), "api": api}


def run_rank(args, rank, world, dist: Dist, backend, extras=None):
    """The rank function of the product run (device agnostic through `backend`): the headline
    workload, then the other metric sizes (`per_config`), each sharded, timed and reduced over
    the ranks in the same way.  `extras(cfg, st, head)` adds keys that need the headline's
    buffers (e2e, the library comparison) before they are freed."""
    cfg = wl.CONFIGS[args.config]
    head, st = run_config(args, cfg, rank, world, dist, backend, steps=args.steps, batch=args.batch)
    solve = cfg.task == "solve"
    more = extras(cfg, st, head) if extras is not None else {}
    del st
    backend.release()
    out = {
        "metric": METRIC_SOLVE if solve else METRIC, "value": head["value"], "unit": head["unit"],
        "n_gpus": world, "steps": head["steps"], "warmup": head["warmup"], "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f32" if cfg.dtype == torch.complex64 else "f64",
        "data": "synthetic (seeded, chunk-keyed; BASELINE.json configs recipe)",
        "config": config_dict(cfg, world, args.scaling, args.batch),
        "roofline": head["roofline"], "roofline_baseline_formula": head["roofline_baseline_formula"],
        "clocks": head["clocks"], "gpu_launches": head["gpu_launches"], "info_nonzero": head["info_nonzero"],
        "e2e": None, "launch": head["launch"], "wall_span_ms": head["wall_span_ms"],
        "batch_per_rank": head["batch_per_rank"], "kernel_ms": head["kernel_ms"],
    }
    out.update(more)
    if args.inv_method != "proposed":
        out["config"]["inv_method"] = args.inv_method + " (SURVEY 8(f) f3: the paper's existing method, not the product path)"
        out.pop("roofline_baseline_formula")
    if cfg.task != "inv":
        out["config"]["task"] = ("solve (1 right-hand side per matrix)" if solve else
                                 "non-Hermitian inversion D^-1 = D*(DD*)^-1")
        out.pop("roofline_baseline_formula", None)
        if cfg.task == "nonherm":
            out["metric"] = "non-Hermitian matrices inverted/sec (SURVEY 8(f) f2, P:135-141), 1 B200"
    # ---- the other metric sizes, each timed the same way on the same ranks
    extra = args.per_config if args.per_config is not None else DEFAULT_PER_CONFIG.get(args.config, "")
    if args.batch is None and args.inv_method == "proposed":
        per = {}
        for tok in [t for t in extra.split(",") if t.strip()]:
            c = wl.CONFIGS[int(tok)]
            res, st = run_config(args, c, rank, world, dist, backend,
                                 steps=min(args.steps, 50) if args.steps else None)
            del st
            backend.release()
            res["workload"] = config_dict(c, world, args.scaling)["workload"]
            res["dtype"] = "f32" if c.dtype == torch.complex64 else "f64"
            per["cfg%d" % c.cid] = res
        if per:
            out["per_config"] = per
            out["gpu_launches"] += sum(r["gpu_launches"] for r in per.values())
            out["gpu_launches_note"] = "headline steps + per_config steps (one kernel launch per step)"
    return out


def run_ours(args, rank, world, local_rank):
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = Dist(world, dev)
    backend = CudaBackend(dev)
    cfg = wl.CONFIGS[args.config]
    if cfg.task == "fxp":
        return run_fxp(args, cfg, rank, world, dev)

    def extras(cfg, st, head):
        more = {}
        if not args.no_e2e and (cfg.task == "solve" or (cfg.task in ("inv", "nonherm")
                                                         and args.inv_method == "proposed")):
            more["e2e"] = e2e_measure(args, cfg, st, world, dist, dev, head["steps"])
        if rank == 0 and world == 1 and not args.no_library:
            more["library_baseline"] = library_baseline(cfg, st["view"], st.get("yview"), dev)
        return more

    out = run_rank(args, rank, world, dist, backend, extras)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, args, budget_s=args.cpu_seconds, dev=dev)
    return out


# ------------------------------------------- f4: fixed-point emulation of the §IV.C study
def run_fxp(args, cfg, rank, world, dev):
    """Times hpdinv_fxp_inv_batched (the proposed method in Q(qm, qf) integer emulation) over
    the cfg8 batch, and reports the study itself: mean relative error of the three methods vs
    the double-precision inverse on a sample of the GPU results (Fig. 1)."""
    import paper_1111_4144_b200 as hp
    start, B, global_batch = shard_plan(cfg, rank, world, args.scaling)
    A, raw = wl.generate_fxp(cfg, start, B, device=dev, seed=args.seed)
    X = torch.empty_like(raw)
    info = torch.empty(B, dtype=torch.int32, device=dev)
    nsat = torch.empty(B, dtype=torch.int64, device=dev)
    steps = args.steps if args.steps is not None else 10
    warmup = max(3, args.warmup)
    dist = Dist(world, dev)
    backend = CudaBackend(dev)
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    ms, _, _ = timed_loop(lambda: hp.fxp_invert(raw, cfg.qm, cfg.qf, "proposed", X, info, nsat),
                          steps, warmup, backend, dist)
    sampler.stop()
    # the study on a sample (host double-precision reference)
    S = min(B, 4096)
    Xr = np.linalg.inv(A[:S].cpu().numpy())
    study = {}
    for method in ("proposed", "eqsolve", "trimat"):
        Xm, im, sm = hp.fxp_invert(raw[:S].contiguous(), cfg.qm, cfg.qf, method)
        torch.cuda.synchronize()
        Xm, im, sm = Xm.cpu().numpy(), im.cpu().numpy(), sm.cpu().numpy()
        ok = (im == 0) & (sm == 0)
        Xf = Xm[..., 0] / 2.0 ** cfg.qf + 1j * Xm[..., 1] / 2.0 ** cfg.qf
        rel = np.linalg.norm((Xf - Xr)[ok], axis=(1, 2)) / np.linalg.norm(Xr[ok], axis=(1, 2))
        Af = A[:S].cpu().numpy()[ok]
        res = np.linalg.norm(Af @ Xf[ok] - np.eye(cfg.n), axis=(1, 2))
        study[method] = {"mean_rel_err": float(rel.mean()), "mean_residual": float(res.mean()),
                         "failures": int((~ok).sum()), "trials": S}
    pk = peaks()
    byts = 2 * 16 * cfg.n * cfg.n * B + 12 * B
    achieved = byts / (ms / 1e3) / 1e9
    out = {
        "metric": "fixed-point Q%d.%d emulated inversions/sec (SURVEY 8(f) f4, P:206-208), 1 B200" % (cfg.qm, cfg.qf),
        "value": global_batch / (ms / 1e3), "unit": "matrices/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "int64 (Q%d.%d raws, 128-bit products)" % (cfg.qm, cfg.qf),
        "data": "synthetic (SPEC.md ensemble, seeded, chunk-keyed)",
        "config": dict(config_dict(cfg, world, args.scaling), task="fxp", format="Q%d.%d" % (cfg.qm, cfg.qf)),
        "roofline": {"bound": "alu", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "kernel": "k_fxp<%d>" % cfg.n, "kernel_ms": ms,
                     "traffic": None, "note": "integer emulation (128-bit software products and "
                     "divisions), ALU bound; the HBM fraction is shown for scale only"},
        "study": study, "clocks": sampler.summary(), "gpu_launches": steps, "e2e": None,
        "e2e_note": "no host-buffer entry point for this task",
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        n0 = 256
        t0 = time.perf_counter()
        oracle.fxp_inv_batched(raw[:n0].cpu().numpy(), cfg.qm, cfg.qf, "proposed")
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": n0 / dt, "unit": "matrices/s", "cores": oracle.max_threads(),
                               "kind": "oracle", "sample": "first %d of the %d matrices of cfg8" % (n0, B)}
    return out


# ------------------------------------------------------- vendor-library comparison (context)
def library_baseline(cfg: wl.Config, view, yview, dev, steps: int = 5):
    """The same workload through PyTorch's batched dense linear algebra on the same GPU
    (cuSOLVER / cuBLAS / MAGMA batched kernels behind torch.linalg): Cholesky + cholesky_inverse
    (the potrf + potri route of SURVEY App. A.3, 'trimat') and, for the solve, cholesky_solve.
    Full Hermitian AoS matrices are formed once outside the timed region.  Context only: it
    is not our kernel and not the reference arm."""
    try:
        B, n = view.shape[0], view.shape[1]
        Af = view.contiguous()
        if cfg.task != "nonherm":
            Af = torch.triu(Af) + torch.triu(Af, 1).conj().transpose(1, 2)
        if cfg.task == "nonherm":
            Af = view.contiguous()

            def run():
                return torch.linalg.inv_ex(Af)[0]
            what = "torch.linalg.inv_ex (batched LU)"
        elif yview is not None:
            y = yview.contiguous().unsqueeze(-1)

            def run():
                L, _ = torch.linalg.cholesky_ex(Af)
                return torch.cholesky_solve(y, L)
            what = "torch.linalg.cholesky_ex + torch.cholesky_solve"
        else:
            def run():
                L, _ = torch.linalg.cholesky_ex(Af)
                return torch.cholesky_inverse(L)
            what = "torch.linalg.cholesky_ex + torch.cholesky_inverse"
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        del Af
        return {"value": B / (ms / 1e3), "unit": UNIT_SOLVE if yview is not None else UNIT, "ms_per_step": ms,
                "what": what + " on full Hermitian AoS matrices, same GPU, %d steps" % steps}
    except Exception as e:  # pragma: no cover - library availability depends on the box
        torch.cuda.synchronize()
        return {"unavailable": repr(e)[:200]}


# ------------------------------------------------------------------- the oracle arm
def oracle_sample(cfg: wl.Config, count: int, seed: int, dev):
    """Host complex128 copy of the first `count` matrices of the workload (exact upcast of
    the bits the GPU consumes when generated on the GPU); fixed-point raws for cfg8."""
    if cfg.task == "fxp":
        return wl.generate_fxp(cfg, 0, count, device=dev, seed=seed)[1].cpu().numpy()
    A = wl.generate(cfg, 0, count, device=dev, seed=seed)
    return A.cpu().to(torch.complex128).numpy()


def oracle_run(cfg: wl.Config, Ah, yh, nthreads: int = 0):
    import oracle
    if cfg.task == "fxp":
        X, info, _ = oracle.fxp_inv_batched(Ah, cfg.qm, cfg.qf, "proposed", nthreads=nthreads)
        return X, info
    if cfg.task == "nonherm":
        return oracle.nonherm_batched(Ah, nthreads=nthreads)
    if cfg.task == "solve":
        return oracle.solve_batched(Ah, yh, cfg.method, nthreads=nthreads)
    return oracle.inv_batched(Ah, cfg.method, nthreads=nthreads)


def oracle_rhs(cfg: wl.Config, count: int, seed: int, dev):
    if cfg.task != "solve":
        return None
    return wl.generate_rhs(cfg, 0, count, device=dev, seed=seed).cpu().to(torch.complex128).numpy()


def cpu_baseline(cfg: wl.Config, args, budget_s: float, dev):
    """The oracle as it stands on the box's host cores (all threads, then 1 thread), on a
    bounded sample of the same workload."""
    import oracle
    oracle.build()
    cores = oracle.max_threads()
    n0 = min(cfg.batch, 1024)
    Ah, yh = oracle_sample(cfg, n0, args.seed, dev), oracle_rhs(cfg, n0, args.seed, dev)
    t0 = time.perf_counter()
    oracle_run(cfg, Ah, yh)
    per = (time.perf_counter() - t0) / Ah.shape[0]
    count = int(min(cfg.batch, max(Ah.shape[0], budget_s / max(per, 1e-9))))
    Ah, yh = oracle_sample(cfg, count, args.seed, dev), oracle_rhs(cfg, count, args.seed, dev)
    t0 = time.perf_counter()
    oracle_run(cfg, Ah, yh)
    dt = time.perf_counter() - t0
    # 1 thread on a sample of ~budget/4 seconds
    c1 = int(max(16, min(count, budget_s / 4.0 / max(per * cores, 1e-9))))
    t1 = time.perf_counter()
    oracle_run(cfg, Ah[:c1], None if yh is None else yh[:c1], nthreads=1)
    dt1 = time.perf_counter() - t1
    return {"value": count / dt, "unit": UNIT_SOLVE if cfg.task == "solve" else UNIT, "cores": cores, "kind": "oracle",
            "sample": "first %d of the %d matrices of cfg%d (%s), fp64 C oracle, OpenMP over matrices"
            % (count, cfg.batch, cfg.cid, cfg.method), "seconds": dt,
            "one_thread": {"value": c1 / dt1, "cores": 1, "sample": "first %d matrices" % c1, "seconds": dt1},
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args, rank, world):
    import oracle
    oracle.build()
    cfg = wl.CONFIGS[args.config]
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    steps = args.steps if args.steps is not None else 5
    warmup = args.warmup if args.warmup is not None else 1
    # each step: a bounded sample sized so the whole run takes ~2-3 minutes
    n0 = min(cfg.batch, 512)
    Ah, yh = oracle_sample(cfg, n0, args.seed, dev), oracle_rhs(cfg, n0, args.seed, dev)
    t0 = time.perf_counter()
    oracle_run(cfg, Ah, yh)
    per = (time.perf_counter() - t0) / Ah.shape[0]
    per_step_s = max(0.2, min(20.0, 150.0 / max(1, steps + warmup)))
    count = int(min(cfg.batch, max(64, per_step_s / max(per, 1e-9))))
    Ah, yh = oracle_sample(cfg, count, args.seed, dev), oracle_rhs(cfg, count, args.seed, dev)
    for _ in range(warmup):
        oracle_run(cfg, Ah, yh)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        X, info = oracle_run(cfg, Ah, yh)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = count / (ms / 1e3)
    cores = oracle.max_threads()
    solve = cfg.task == "solve"
    UNITX = UNIT_SOLVE if solve else UNIT
    return {
        "impl": "reference", "metric": METRIC_SOLVE if solve else METRIC, "value": value, "unit": UNITX,
        "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, chunk-keyed; BASELINE.json configs recipe)",
        "config": config_dict(cfg, world, args.scaling, args.batch),
        "sample_per_step": count,
        "cpu_baseline": {"value": value, "unit": UNITX, "cores": cores, "kind": "oracle",
                         "sample": "first %d of the %d matrices of cfg%d per step" % (count, cfg.batch, cfg.cid),
                         "cpu": _cpu_model()},
        "e2e": {"value": value, "unit": UNITX, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "info_nonzero": int((info != 0).sum()),
    }


# ------------------------------------------------------------------- launcher
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(nproc: int, argv) -> int:
    """Re-launch this script under torch.distributed.run with one rank per GPU (the driver's
    own launch line); returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        return spawn_ranks(args.gpus, argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return 0
        print(json.dumps(run_reference(args, rank, world)), flush=True)
        return 0
    if world != args.gpus:
        print("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world), file=sys.stderr)
        return 2
    if world > 1:
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
