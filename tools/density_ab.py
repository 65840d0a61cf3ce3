#!/usr/bin/env python3
"""A/B of the dense-step GEMM launches in the density view: device time of one density range
with the GEMM launches (default) and with the same steps as dataflow tiles (QCG_NO_GEMM=1).
  python tools/density_ab.py <stem> [passes]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

if len(sys.argv) > 3:  # child: one engine, one range
    from conftest import payload_path
    from paper_2010_14962_b200 import Engine
    stem, passes = sys.argv[1], int(sys.argv[2])
    with Engine(payload_path(stem), device=0, mode="density") as e:
        st = e.plan_stats()
        n = passes << st["batch_bits"]
        lo = 0
        e.sum_range(lo, lo + n)  # warm-up
        v = e.sum_range(lo, lo + n)
        ms = e.last_run()["device_ms"]
        kinds = {}
        for p in e.profile_pass(lo, lo + (1 << st["batch_bits"])):
            kinds[p["kind"]] = kinds.get(p["kind"], 0.0) + p["ms"]
    print(f"{sys.argv[3]:8s} {stem} batch_bits={st['batch_bits']} passes={passes} device_ms={ms:.3f} value={v:.12g} "
          + " ".join(f"{k}={t:.3f}ms" for k, t in sorted(kinds.items(), key=lambda x: -x[1])))
else:
    stem = sys.argv[1]
    passes = sys.argv[2] if len(sys.argv) > 2 else "2"
    for tag, env in (("gemm", {}), ("no-gemm", {"QCG_NO_GEMM": "1"})):
        subprocess.run([sys.executable, __file__, stem, passes, tag], env={**os.environ, **env}, check=False)
