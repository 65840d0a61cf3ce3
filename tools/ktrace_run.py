#!/usr/bin/env python3
"""In-graph timeline of one pass (QCG_KTRACE build of the engine: make EXTRA=-DQCG_KTRACE OUT=...):
  QCUT_GPU_LIB=build_var/ktrace/libqcut_gpu.so python tools/ktrace_run.py <stem> 2> trace.txt
The engine prints, after every call, CTA (0,0) of every kernel: start, dependency-wait done, end (ns)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import payload_path  # noqa: E402
from paper_2010_14962_b200 import Engine  # noqa: E402

with Engine(payload_path(sys.argv[1]), device=0, mode="ket") as e:
    n = 2 ** e.plan_stats()["n_cut"]
    for _ in range(5):
        e.bench_cold(1, 0, n)
