#!/usr/bin/env python3
"""Summarise an ncu launch list (gpu__time_duration.sum) per kernel name; optional last-N window."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
hdr = None
ts = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            ts.append((d["Kernel Name"].split("(")[0], float(d["Metric Value"]), d["Grid Size"], d["Block Size"]))
if last:
    ts = ts[-last:]
tot = sum(t for _, t, _, _ in ts)
print(f"launches {len(ts)}  total {tot/1e3:.1f} us")
agg = defaultdict(lambda: [0, 0.0])
for n, t, _, _ in ts:
    agg[n][0] += 1
    agg[n][1] += t
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {n:40s} n={c:5d}  {t/1e3:9.1f} us  {100*t/tot:5.1f}%")
print("top launches:")
for n, t, g, b in sorted(ts, key=lambda x: -x[1])[:12]:
    print(f"  {n:40s} {t/1e3:9.1f} us grid={g} block={b}")
