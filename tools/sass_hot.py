#!/usr/bin/env python
"""Hot spots of an ncu source page (SASS): opcode histogram of executed warp instructions and of
stall samples, and the hottest address ranges.  Usage: ncu -i rep --page source --csv
--print-source sass > s.csv; python tools/sass_hot.py s.csv [nranges]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
ins = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        ex = float(r[ix["Instructions Executed"]] or 0)
        smp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    op = r[ix["Source"]].strip().split()
    op = [o for o in op if not o.startswith("@")]
    ins.append((int(r[ix["Address"]], 16) if r[ix["Address"]].startswith("0x") else int(r[ix["Address"]] or 0),
                op[0] if op else "?", ex, smp, r[ix["Source"]].strip()))
tot_ex = sum(i[2] for i in ins)
tot_s = sum(i[3] for i in ins)
by_op = collections.defaultdict(lambda: [0.0, 0.0])
for a, op, ex, smp, src in ins:
    by_op[op.split(".")[0]][0] += ex
    by_op[op.split(".")[0]][1] += smp
print("total warp instructions %.4g, samples %.4g, static instructions %d" % (tot_ex, tot_s, len(ins)))
print("%-12s %10s %7s %7s" % ("opcode", "executed", "%exec", "%samp"))
for op, (ex, smp) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:25]:
    print("%-12s %10.4g %6.1f%% %6.1f%%" % (op, ex, 100 * ex / tot_ex, 100 * smp / max(tot_s, 1)))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if n:
    # contiguous ranges of 64 instructions, hottest by samples
    rng = collections.defaultdict(lambda: [0.0, 0.0])
    for k, (a, op, ex, smp, src) in enumerate(ins):
        rng[k // 64][0] += ex
        rng[k // 64][1] += smp
    print("hottest 64-instruction ranges (index: executed, samples)")
    for k, (ex, smp) in sorted(rng.items(), key=lambda kv: -kv[1][1])[:n]:
        print("  [%5d..%5d] %10.4g %6.1f%%" % (k * 64, k * 64 + 63, ex, 100 * smp / max(tot_s, 1)))
