#!/usr/bin/env python
"""Aggregate an ncu source page (--print-source cuda,sass) per CUDA source line:
warp-level instructions executed and stall samples, top lines first.

    python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, line, src = None, None, None
agg = {}
hdr = None
tot_i = tot_s = 0
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].rsplit("/", 1)[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(row) < len(hdr) // 2:
        continue
    if row[0]:
        line, src = row[0], row[1]
        continue
    if row[2] in ("...", "-", ""):
        continue
    try:
        n = int(float(row[ii]))
        s = int(float(row[si]))
    except ValueError:
        continue
    k = (fname, line)
    a = agg.setdefault(k, [0, 0, src])
    a[0] += n
    a[1] += s
    tot_i += n
    tot_s += s
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
for (f, l), (n, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{n:>11} {100*n/max(1,tot_i):5.1f}%i {100*s/max(1,tot_s):5.1f}%s {f}:{l:<5} {src.strip()[:90]}")
