#!/usr/bin/env python
"""Print the last step of an ncu launch list (gpu__time_duration.sum csv): one line per kernel launch."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; rows = rows[1:]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tot = 0
for r in rows[-n:]:
    v = float(r[vi].replace(',', '')) / 1000
    tot += v
    print(f"{v:9.1f} us  {r[ki][:90]}")
print(f"{tot:9.1f} us total (last {n})")
