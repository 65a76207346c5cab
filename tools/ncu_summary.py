#!/usr/bin/env python
"""Summarise an ncu --set full report (one or more kernels) into a short text table.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [out.txt] [--traffic cfgK batch k_family<c64,chol>]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe inst %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU inst %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs), blocks"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "instructions (warp)"),
]


def load(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
        kernels.append(d)
    return kernels


def main():
    rep = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
    lines = []
    for d in load(rep):
        lines.append("kernel: %s" % d.get("Kernel Name", ("", "?"))[1])
        for k, label in KEYS:
            if k in d:
                u, v = d[k]
                lines.append("  %-34s %16s %s   [%s]" % (label, v, u, k))
        stalls = sorted(((float(v.replace(",", "")), h) for h, (u, v) in d.items()
                         if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio")
                         and v not in ("", "n/a")), reverse=True)[:6]
        for v, h in stalls:
            lines.append("  stall %-40s %8.2f" % (h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), v))
        lines.append("")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write("# ncu --set full summary of %s\n%s\n" % (os.path.basename(rep), text))
    if "--traffic" in sys.argv:
        i = sys.argv.index("--traffic")
        cfg, batch, short = sys.argv[i + 1], int(sys.argv[i + 2]), sys.argv[i + 3]
        d = load(rep)[0]
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tb = sum(float(d[k][1].replace(",", "")) * mult[d[k][0]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
        t = json.load(open(path)) if os.path.exists(path) else {}
        name = d["Kernel Name"][1]
        t[cfg] = {"kernel_full": name, "kernel": short, "batch": batch, "dram_bytes_per_launch": tb, "source": os.path.basename(rep)}
        json.dump(t, open(path, "w"), indent=1)
        print("traffic", cfg, tb)


if __name__ == "__main__":
    main()
