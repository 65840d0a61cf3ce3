#!/usr/bin/env python3
"""Device time per amplitude of arbitrary payloads (ket view, all slices per call):
    python tools/time_payload.py a.json b.json.gz ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_14962_b200 import Engine  # noqa: E402

for path in sys.argv[1:]:
    with Engine(path, device=0, mode="ket") as e:
        st = e.plan_stats()
        a = e.ket_sum()
        e.bench(5)
        r = e.bench(20)
        ms = sorted(r["pass_ms"])[len(r["pass_ms"]) // 2] * st["chunks"]
        print(f"{os.path.basename(path)}: {ms:.4f} ms/amplitude  peak {st['peak_rank']}  b {st['batch_bits']}  "
              f"passes {st['chunks']}  moved {st['moved_bytes']:.3g} B  arena {st['arena_bytes']:.3g} B  |A|^2 {abs(a)**2:.6e}",
              flush=True)
