#!/usr/bin/env python3
"""Per-launch device times of one pass (CUDA events, qc_engine_profile_pass) with achieved
HBM GB/s and FP64 TFLOP/s per launch:  python tools/launch_profile.py --config cfg4os"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, payload  # noqa: E402
from paper_2010_14962_b200 import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
e = Engine(payload(CONFIGS[a.config]["stem"]), device=0, mode="ket")
st = e.plan_stats()
n = 1 << st["batch_bits"]
e.ket_sum(0, n)
rows = e.profile_pass(0, n)
tot = sum(r["ms"] for r in rows)
print(f"{a.config}: pass {tot:.3f} ms, {len(rows)} launches, batch_bits {st['batch_bits']}, passes {st['chunks']}")
for i, r in sorted(enumerate(rows), key=lambda x: -x[1]["ms"])[: a.top]:
    gbs = r["bytes"] / r["ms"] / 1e6 if r["ms"] > 0 else 0
    tfs = r["exec_flops"] / r["ms"] / 1e9 if r["ms"] > 0 else 0
    print(f"  [{i:3d}] {r['kind']:7s} {r['ms']:9.3f} ms {100 * r['ms'] / tot:5.1f}%  {r['bytes'] / 1e9:9.3f} GB "
          f"{gbs:7.0f} GB/s  {tfs:6.2f} TF/s  n={r.get('n', '')}")
print(e.describe())
# critical path through the launch DAG (deps from describe), weighted by the measured times
import re  # noqa: E402

deps = {}
for line in e.describe().split("\n"):
    m = re.match(r"\s+\[(\d+)\] \w+ .*?(?:deps=([\d,]+))?(?: |$)", line)
    if m and "steps=" in line:
        dm = re.search(r"deps=([\d,]+)", line)
        deps[int(m.group(1))] = [int(x) for x in dm.group(1).split(",") if x] if dm else []
fin, prev = {}, {}
for i in range(len(rows)):
    best, arg = 0.0, None
    for dpn in deps.get(i, []):
        if fin.get(dpn, 0.0) > best:
            best, arg = fin[dpn], dpn
    fin[i] = best + rows[i]["ms"]
    prev[i] = arg
end = max(fin, key=fin.get)
path = []
while end is not None:
    path.append(end)
    end = prev[end]
path.reverse()
print(f"critical path {fin[path[-1]]:.3f} ms of {tot:.3f} ms serial: " +
      " -> ".join(f"[{i}] {rows[i]['kind']} {1e3 * rows[i]['ms']:.0f}us" for i in path))
