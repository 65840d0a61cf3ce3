#!/usr/bin/env python3
"""Run engine passes for ncu: one warm-up pass, then `--passes` passes.

  ncu --set full -k regex:k_step --launch-skip <warm k_step launches + dominant> --launch-count 1 \
      python tools/profile_pass.py --config cfg2
Prints the dominant kernel index and the skip count to use.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, payload  # noqa: E402
from paper_2010_14962_b200 import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--passes", type=int, default=1)
ap.add_argument("--mode", default="ket")
ap.add_argument("--slices", type=int, default=0, help="ket slices per call (default: all)")
a = ap.parse_args()
e = Engine(payload(CONFIGS[a.config]["stem"]), device=0, mode=a.mode)
st = e.plan_stats()
n_steps = st["n_steps"]
print(f"dominant_kernel={st['dominant_kernel']} bytes={st['dominant_bytes']:.4g} "
      f"skip_for_second_pass={n_steps + st['dominant_kernel']}", flush=True)
for _ in range(1 + a.passes):
    if a.slices:
        v = e.ket_sum(0, a.slices)
    else:
        v = e.ket_sum() if a.mode == "ket" else e.run_serial()
print("value", v, e.last_run())
