#!/usr/bin/env python3
"""Rank candidate payloads by the engine's own host planner (no GPU needed): bytes the
engine's kernels move per amplitude (after its fusions), arena size and launch count.
The searches' byte model counts every intermediate; the engine keeps fused intermediates
on chip, so its count is the one that tracks measured time.
    python tools/rerank_plans.py cand1.json cand2.json ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_14962_b200 import Engine  # noqa: E402


def engine_cost(path, budget=100 << 30):
    with Engine(path, device=-1, mode="ket", mem_budget_bytes=budget) as e:
        st = e.plan_stats()
    return st["moved_bytes"], st


if __name__ == "__main__":
    rows = []
    for p in sys.argv[1:]:
        mb, st = engine_cost(p)
        rows.append((mb, p, st))
    for mb, p, st in sorted(rows, key=lambda r: r[0]):
        print(f"{mb:.4g} B moved  arena {st['arena_bytes']:.3g} B  launches {st['n_kernels']}  peak {st['peak_rank']}  {p}")
