#!/usr/bin/env python
"""bench.py -- throughput of the batched HPD inversion hot path (BASELINE.json metric).

One step = one pass of the whole hot path (load upper(A) -> Cholesky/LDL -> proposed
inversion -> mirror -> store) over one batch of synthetic matrices, i.e.
one call of the C ABI entry point.  Default workload: BASELINE.json configs[1] (cfg2: 2^20
complex64 8x8 HPD matrices, interleaved layout) on N=1 GPU.  `--config k` selects another.

Multi-GPU (torchrun, one process per GPU): every rank inverts its own slice of a global
batch of N x B matrices generated locally from chunk-keyed seeds (weak scaling, no data-path
collective).  Timing: CUDA events on the launching stream between a barrier +
synchronize on both sides; the max over ranks is reported.

`--impl reference` times the fp64 CPU oracle (the reference arm of this tier) on bounded
samples of the same workload, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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
L2_BYTES = 126 * 2**20
SMS = 148


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, default=2, choices=sorted(wl.CONFIGS))
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-library", action="store_true", help="skip the vendor-library comparison")
    p.add_argument("--batch", type=int, default=None,
                   help="override the config's per-GPU batch (e.g. an L2-resident study; not a BASELINE line)")
    p.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                   help="replay each step from a CUDA graph (auto: for launch-bound batches, cfg1)")
    p.add_argument("--inv-method", choices=["proposed", "eqsolve", "trimat"], default="proposed",
                   help="SURVEY 8(f) f3: time one of the paper's existing methods on the GPU instead")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    return p.parse_args()


# ----------------------------------------------------------------------------- helpers
METRIC_SOLVE = "HPD linear systems solved/sec (SURVEY 8(f) f1: A x = y, eqs. 5-7 / 12-14), 1 B200"
UNIT_SOLVE = "systems/s"


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
    """FP32 / FP64 FMA peak from unit counts: 148 SMs x {128, 64} FMA/clk x 2."""
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


def load_traffic(cfg: wl.Config, kernel: str):
    """Per-launch DRAM bytes of this kernel from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        t = json.load(open(path))
        rec = t.get("cfg%d" % cfg.cid)
        if rec and rec.get("kernel") == kernel and rec.get("batch") == cfg.batch:
            return float(rec["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


# ------------------------------------------------------------------------------ ours
def run_ours(args, rank, world, local_rank):
    import paper_1111_4144_b200 as hp

    cfg = wl.CONFIGS[args.config]
    if args.batch:
        import dataclasses
        cfg = dataclasses.replace(cfg, batch=int(args.batch))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    B = cfg.batch
    if cfg.task == "fxp":
        return run_fxp(args, cfg, rank, world, dev)
    A = wl.generate(cfg, rank * B, B, device=dev, seed=args.seed)   # this rank's slice
    store, view = wl.to_layout(A, cfg.layout)
    del A
    info = torch.empty(B, dtype=torch.int32, device=dev)
    solve = cfg.task == "solve"
    metric, unit = (METRIC_SOLVE, UNIT_SOLVE) if solve else (METRIC, UNIT)
    if solve:
        Y = wl.generate_rhs(cfg, rank * B, B, device=dev, seed=args.seed)
        ystore, yview = wl.vec_layout(Y, cfg.layout)
        del Y
        Xv = torch.empty_strided(yview.shape, yview.stride(), dtype=cfg.dtype, device=dev)
        kernel = hp.solve_kernel_name(cfg.method, cfg.dtype, cfg.n)

        def step():
            hp.solve(view, yview, cfg.method, Xv=Xv, info=info)
    elif cfg.task == "nonherm":
        X = wl.empty_like_layout(view)
        kernel = hp.nonherm_kernel_name(cfg.dtype, cfg.n)

        def step():
            hp.invert_nonhermitian(view, Dinv=X, info=info)
    elif args.inv_method != "proposed":
        X = wl.empty_like_layout(view)
        kernel = hp.method_kernel_name(args.inv_method, cfg.dtype, cfg.n)

        def step():
            hp.invert_method(view, args.inv_method, X=X, info=info)
    else:
        X = wl.empty_like_layout(view)
        kernel = hp.kernel_name(cfg.method, cfg.dtype, B, cfg.n, (view.stride(0), view.stride(2)))

        def step():
            hp.invert(view, cfg.method, X=X, info=info)

    per_step_guess = algorithmic_bytes(cfg) * B / 6.0e12
    steps = args.steps if args.steps is not None else max(20, min(2000, int(0.5 / per_step_guess)))
    warmup = max(3, args.warmup)

    def barrier():
        if world > 1:
            torch.distributed.barrier(device_ids=[local_rank])

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    bad = int((info != 0).sum().item())
    # launch-bound batches (cfg1: 1024 matrices, a few µs of GPU work) replay the step from a CUDA
    # graph so the host-side Python/ctypes overhead does not pose as kernel time
    use_graph = args.graph == "on" or (args.graph == "auto" and algorithmic_bytes(cfg) * B < 64 * 2**20)
    launch = "direct C-ABI call per step"
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        torch.cuda.synchronize()
        step = graph.replay
        launch = "CUDA graph of the C-ABI call (one kernel node), replayed per step"
    barrier()
    torch.cuda.synchronize()

    sampler = ClockSampler(torch.cuda.current_device())
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    sampler.start()
    t0.record(stream)
    for k in range(steps):
        evs[k][0].record(stream)
        step()
        evs[k][1].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    sampler.stop()
    barrier()
    elapsed_ms = t0.elapsed_time(t1)
    kern_ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    t = torch.tensor([elapsed_ms, kern_ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    elapsed_ms, kern_ms = t.tolist()
    ms_per_step = elapsed_ms / steps
    value = world * B / (ms_per_step / 1e3)

    # ---- end to end through the host-buffer C entry point (H2D + kernel + D2H timed)
    e2e = None
    if not args.no_e2e and solve:
        # the solve end to end through hpdinv_solve_host (pinned host A, y -> x)
        A_host = store.cpu().pin_memory()
        Y_host = ystore.cpu().pin_memory()
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
        chunk = max(4096, B // 8)
        ws = torch.empty(hp.solve_host_workspace_bytes(cfg.dtype, cfg.n, chunk), dtype=torch.uint8, device=dev)
        e2e_steps = max(3, min(steps, 10))
        for _ in range(2):
            hp.solve_host(vh, yh, cfg.method, xh, info_h, ws, chunk)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(e2e_steps):
            hp.solve_host(vh, yh, cfg.method, xh, info_h, ws, chunk)
        b.record(stream)
        torch.cuda.synchronize()
        barrier()
        te = torch.tensor([a.elapsed_time(b) / e2e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        same = torch.equal(xh.contiguous(), Xv.cpu().contiguous()) and torch.equal(info_h, info.cpu())
        e2e = {"value": world * B / (te.item() / 1e3), "unit": UNIT_SOLVE, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(cfg.elem_bytes * cfg.n * B + 4 * B), "ms_per_step": te.item(),
               "chunk": chunk, "matches_device_run": bool(same), "api": "hpdinv_solve_host (pinned host buffers)"}
    if not args.no_e2e and cfg.task in ("inv", "nonherm") and args.inv_method == "proposed":
        nh = cfg.task == "nonherm"
        A_host = store.cpu().pin_memory()
        if cfg.layout == "soa":
            vh = wl.soa_view(A_host, B, cfg.n)
            X_host = torch.empty_like(A_host).pin_memory()
            xh = wl.soa_view(X_host, B, cfg.n)
            h2d = cfg.elem_bytes * (cfg.n * cfg.n if nh else cfg.n * (cfg.n + 1) // 2) * B
        else:
            vh = A_host
            X_host = torch.empty_like(A_host).pin_memory()
            xh = X_host
            h2d = cfg.elem_bytes * cfg.n * cfg.n * B
        info_h = torch.empty(B, dtype=torch.int32).pin_memory()
        chunk = max(4096, B // 8)
        ws = torch.empty(hp.host_workspace_bytes(cfg.dtype, cfg.n, chunk), dtype=torch.uint8, device=dev)
        e2e_steps = max(3, min(steps, 10))
        hmethod = "nonherm" if nh else cfg.method
        for _ in range(2):
            hp.invert_host(vh, hmethod, xh, info_h, ws, chunk)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(e2e_steps):
            hp.invert_host(vh, hmethod, xh, info_h, ws, chunk)
        b.record(stream)
        torch.cuda.synchronize()
        barrier()
        te = torch.tensor([a.elapsed_time(b) / e2e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        # the result read back must match the device-resident run bit for bit
        same = torch.equal(xh.contiguous(), X.cpu().contiguous()) and torch.equal(info_h, info.cpu())
        e2e = {"value": world * B / (te.item() / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(cfg.elem_bytes * cfg.n * cfg.n * B + 4 * B),
               "ms_per_step": te.item(), "chunk": chunk, "matches_device_run": bool(same),
               "api": "hpdinv_inv_host (pinned host buffers)"}

    # ---- roofline of the (single) kernel of the step
    pk = peaks()
    clocks = sampler.summary()
    bytes_launch = algorithmic_bytes(cfg) * B
    mem_s = bytes_launch / (pk["hbm_gbs"] * 1e9)
    fp_tf = fp_peak_tflops(cfg.dtype, pk["sm_max_mhz"])
    flops_launch = 8.0 * cmul_per_matrix(cfg.n, cfg.task) * B
    fp_s = flops_launch / (fp_tf * 1e12)
    if fp_s > mem_s:
        achieved = flops_launch / (kern_ms / 1e3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": fp_tf, "unit": "TFLOP/s",
                "frac": achieved / fp_tf, "peak_source": "derived: 148 SMs x %d FMA/clk x 2 x %.0f MHz"
                % (128 if cfg.dtype == torch.complex64 else 64, pk["sm_max_mhz"])}
    else:
        achieved = bytes_launch / (kern_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "peak_source": pk["source"]}
    roof["traffic"] = load_traffic(cfg, kernel)
    roof["algorithmic_bytes_per_launch"] = bytes_launch
    roof["kernel"] = kernel
    roof["kernel_ms"] = kern_ms
    # BASELINE.json's own formula: max(16 N^2 batch / HBM, multiply count / FP peak)
    bj_bytes = 2 * cfg.elem_bytes * cfg.n ** 2 * B
    bj_t = max(bj_bytes / (pk["hbm_gbs"] * 1e9), fp_s)
    out = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if cfg.dtype == torch.complex64 else "f64",
        "data": "synthetic (seeded, chunk-keyed; BASELINE.json configs recipe)",
        "config": {"workload": "cfg%d: %s" % (cfg.cid, cfg.desc), "n": cfg.n,
                   "batch_per_gpu": B, "global_batch": world * B,
                   "elem": "complex64" if cfg.dtype == torch.complex64 else "complex128",
                   "method": cfg.method, "layout": cfg.layout,
                   "parallelism": "batch slices, %d rank(s), no collective" % world, "launch": launch,
                   "l2": "inputs larger than L2 (%.0f MB working set > 126 MB); no flush"
                   % ((bj_bytes) / 1e6) if bj_bytes > L2_BYTES else "working set fits L2"},
        "roofline": roof,
        "roofline_baseline_formula": {"time_s": bj_t, "frac": bj_t / (kern_ms / 1e3),
                                      "bytes": bj_bytes, "note": "BASELINE.json north_star formula"},
        "clocks": clocks, "gpu_launches": steps, "info_nonzero": bad, "e2e": e2e,
    }
    if args.inv_method != "proposed":
        out["config"]["inv_method"] = args.inv_method + " (SURVEY 8(f) f3: the paper's existing method, not the product path)"
        out.pop("roofline_baseline_formula")
    if cfg.task != "inv":
        out["config"]["task"] = ("solve (1 right-hand side per matrix)" if solve else
                                 "non-Hermitian inversion D^-1 = D*(DD*)^-1")
        out.pop("roofline_baseline_formula", None)
        if e2e is None:
            out["e2e_note"] = "no host-buffer entry point for this task yet"
        if cfg.task == "nonherm":
            out["metric"] = "non-Hermitian matrices inverted/sec (SURVEY 8(f) f2, P:135-141), 1 B200"
    if rank == 0 and world == 1 and not args.no_library:
        out["library_baseline"] = library_baseline(cfg, view, yview if solve else None, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, args, budget_s=args.cpu_seconds, dev=dev)
    return out


# ------------------------------------------- f4: fixed-point emulation of the §IV.C study
def run_fxp(args, cfg, rank, world, dev):
    """Times hpdinv_fxp_inv_batched (the proposed method in Q(qm, qf) integer emulation) over
    the cfg8 batch, and reports the study itself: mean relative error of the three methods vs
    the double-precision inverse on a sample of the GPU results (Fig. 1)."""
    import paper_1111_4144_b200 as hp
    B = cfg.batch
    A, raw = wl.generate_fxp(cfg, rank * B, B, device=dev, seed=args.seed)
    X = torch.empty_like(raw)
    info = torch.empty(B, dtype=torch.int32, device=dev)
    nsat = torch.empty(B, dtype=torch.int64, device=dev)
    steps = args.steps if args.steps is not None else 10
    warmup = max(3, args.warmup)
    for _ in range(warmup):
        hp.fxp_invert(raw, cfg.qm, cfg.qf, "proposed", X, info, nsat)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier(device_ids=[dev.index])
    sampler = ClockSampler(torch.cuda.current_device())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler.start()
    a.record()
    for _ in range(steps):
        hp.fxp_invert(raw, cfg.qm, cfg.qf, "proposed", X, info, nsat)
    b.record()
    torch.cuda.synchronize()
    sampler.stop()
    t = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = t.item()
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
        "value": world * B / (ms / 1e3), "unit": "matrices/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64 (Q%d.%d raws, 128-bit products)" % (cfg.qm, cfg.qf),
        "data": "synthetic (SPEC.md ensemble, seeded, chunk-keyed)",
        "config": {"workload": "cfg%d: %s" % (cfg.cid, cfg.desc), "n": cfg.n, "batch_per_gpu": B,
                   "task": "fxp", "format": "Q%d.%d" % (cfg.qm, cfg.qf),
                   "l2": "inputs larger than L2" if byts > L2_BYTES else "working set fits L2"},
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


def oracle_run(cfg: wl.Config, Ah, yh):
    import oracle
    if cfg.task == "fxp":
        X, info, _ = oracle.fxp_inv_batched(Ah, cfg.qm, cfg.qf, "proposed")
        return X, info
    if cfg.task == "nonherm":
        return oracle.nonherm_batched(Ah)
    if cfg.task == "solve":
        return oracle.solve_batched(Ah, yh, cfg.method)
    return oracle.inv_batched(Ah, cfg.method)


def oracle_rhs(cfg: wl.Config, count: int, seed: int, dev):
    if cfg.task != "solve":
        return None
    return wl.generate_rhs(cfg, 0, count, device=dev, seed=seed).cpu().to(torch.complex128).numpy()


def cpu_baseline(cfg: wl.Config, args, budget_s: float, dev):
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
    return {"value": count / dt, "unit": UNIT_SOLVE if cfg.task == "solve" else UNIT, "cores": cores, "kind": "oracle",
            "sample": "first %d of the %d matrices of cfg%d (%s), fp64 C oracle, OpenMP over matrices"
            % (count, cfg.batch, cfg.cid, cfg.method), "seconds": dt,
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
        "impl": "reference", "metric": METRIC_SOLVE if solve else METRIC, "value": value, "unit": UNITX, "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg%d: %s" % (cfg.cid, cfg.desc), "n": cfg.n,
                   "batch_per_gpu": cfg.batch, "method": cfg.method, "layout": cfg.layout,
                   "sample_per_step": count},
        "cpu_baseline": {"value": value, "unit": UNITX, "cores": cores, "kind": "oracle",
                         "sample": "first %d of the %d matrices of cfg%d per step" % (count, cfg.batch, cfg.cid),
                         "cpu": _cpu_model()},
        "e2e": {"value": value, "unit": UNITX, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "info_nonzero": int((info != 0).sum()),
    }


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return 0
        print(json.dumps(run_reference(args, rank, world)), flush=True)
        return 0
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
