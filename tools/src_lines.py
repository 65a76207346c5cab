#!/usr/bin/env python
"""Per-source-line totals (instructions executed, stall samples) from an ncu source page printed
with --print-source cuda,sass.  Usage: python tools/src_lines.py page.csv [file-substring] [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur_file = None
hdr = None
lines = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] and r[0].isdigit():          # a CUDA line with its aggregated metrics
        try:
            ex = float(r[hdr.index("Instructions Executed")] or 0)
            smp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        if want in (cur_file or ""):
            lines[(cur_file.split("/")[-1], int(r[0]))] = (ex, smp, r[1].strip()[:90])
tot_e = sum(v[0] for v in lines.values()) or 1
tot_s = sum(v[1] for v in lines.values()) or 1
print("lines with metrics: %d, executed %.4g, samples %.4g" % (len(lines), tot_e, tot_s))
for k, (ex, smp, src) in sorted(lines.items(), key=lambda kv: -kv[1][1])[:top]:
    print("%-14s %4d %6.1f%%ex %6.1f%%smp  %s" % (k[0], k[1], 100 * ex / tot_e, 100 * smp / tot_s, src))
