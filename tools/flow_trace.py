#!/usr/bin/env python3
"""Latency anatomy of the dataflow executor (k_flow) from a QCG_FLOW_TRACE capture.

  QCG_FLOW_TRACE=/tmp/t.bin python tools/flow_trace.py --config cfg5bt      # capture + report
  python tools/flow_trace.py --file /tmp/t.bin                              # report only

Per flow launch: span, per-item phase times (pick->deps ready, operand loads,
compute+store+release), gaps between a CTA's consecutive items, continuation share, and a
critical path walked back from the last item (each item's predecessor = the item that
finished last before it became ready).
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def read(path):
    raw = open(path, "rb").read()
    recs, pos = [], 0
    while pos < len(raw):
        n, nl, nstatic = np.frombuffer(raw, np.uint64, 3, pos)
        pos += 24
        offs = np.frombuffer(raw, np.uint64, int(nl), pos).astype(np.int64)
        pos += 8 * int(nl)
        t = np.frombuffer(raw, np.uint64, 8 * int(n), pos).reshape(-1, 8).astype(np.int64)
        pos += 64 * int(n)
        recs.append((offs, t, int(nstatic)))
    return recs[-1]


def report(offs, t, nstatic):
    bounds = list(offs) + [len(t)]
    for L in range(len(offs)):
        r = t[bounds[L]:bounds[L + 1]]
        r = r[r[:, 1] > 0]
        if len(r) == 0:
            continue
        step = r[:, 0] >> 32
        cont = r[:, 0] & 1
        t0, t1, t2, t4 = r[:, 1], r[:, 2], r[:, 3], r[:, 4]
        w0lat = (t1 >> 40) & 0xffff
        wslow = (t1 >> 56) & 0xff
        t1 = (t1 & 0xffffffffff) | (t0 & ~0xffffffffff)
        cta = (r[:, 0] >> 8) & 255  # SM id
        base = t0.min()
        span = (t4.max() - base) / 1e3
        print(f"flow launch {L}: {len(r)} items, {len(set(step.tolist()))} steps, span {span:.1f} us, "
              f"continuations {cont.sum()} ({100 * cont.mean():.0f}%), CTAs used {len(set(cta.tolist()))}")
        for name, v in (("ready wait", t1 - t0), ("loads", t2 - t1), ("compute+store+release", t4 - t2),
                        ("item total", t4 - t0)):
            print(f"   {name:22s} median {np.median(v) / 1e3:6.2f} us  p90 {np.percentile(v, 90) / 1e3:6.2f} us")
        # gaps between consecutive items of a CTA
        gaps = []
        for c in set(cta.tolist()):
            idx = np.flatnonzero(cta == c)
            o = idx[np.argsort(t0[idx])]
            gaps += list((t0[o[1:]] - t4[o[:-1]]) / 1e3)
        if gaps:
            print(f"   CTA gap between items   median {np.median(gaps):6.2f} us  p90 {np.percentile(gaps, 90):6.2f} us")
        # critical path: walk back from the last finisher
        order = np.argsort(t4)
        i = int(np.argmax(t4))
        path = []
        while True:
            path.append(i)
            ready = t1[i]
            prev = order[t4[order] < ready]
            if len(prev) == 0:
                break
            j = int(prev[-1])
            if j == i or t4[j] < base:
                break
            i = j
        path = path[::-1]
        nta, ntb = (r[:, 0] >> 16) & 255, (r[:, 0] >> 24) & 255
        slow = np.argsort(t2 - t1)[::-1][:8]
        print("   slowest loads (step nTA nTB us): " + " ".join(
            f"({step[k]} {nta[k]} {ntb[k]} {(t2[k] - t1[k]) / 1e3:.1f} dbg nd={r[k, 5] & 255} q={(r[k, 5] >> 8) & 0xffff} "
            f"seen={(r[k, 5] >> 24) & 0xffff} need={(r[k, 5] >> 40) & 0xffff} A@{r[k, 6]}{'s' if r[k, 6] < nstatic else ''} "
            ")" for k in slow) + f"  [static < {nstatic}]")
        fast = np.argsort(t2 - t1)[:4]
        print("   fastest loads: " + " ".join(
            f"({step[k]} {nta[k]} {ntb[k]} {(t2[k] - t1[k]) / 1e3:.1f} A@{r[k, 6]} B@{r[k, 7]})" for k in fast))
        print(f"   critical path ~{len(path)} items: " + " ".join(
            f"[{(t0[k] - base) / 1e3:.1f}+{(t1[k] - t0[k]) / 1e3:.1f}/{(t2[k] - t1[k]) / 1e3:.1f}/"
            f"{(t4[k] - t2[k]) / 1e3:.1f}{'c' if cont[k] else ''}]" for k in path[:40]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config")
    ap.add_argument("--file", default=os.environ.get("QCG_FLOW_TRACE", "/tmp/qcg_flow_trace.bin"))
    a = ap.parse_args()
    if a.config:
        os.environ["QCG_FLOW_TRACE"] = a.file
        if os.path.exists(a.file):
            os.unlink(a.file)
        from bench import CONFIGS, payload
        from paper_2010_14962_b200 import Engine

        e = Engine(payload(CONFIGS[a.config]["stem"]), device=0, mode="ket")
        n = 1 << e.plan_stats()["batch_bits"]
        for _ in range(3):
            e.ket_sum(0, n)
        e.close()
    report(*read(a.file))


if __name__ == "__main__":
    main()


def steps_timeline(path, launch, steps):
    offs, t, nstatic = read(path)
    bounds = list(offs) + [len(t)]
    r = t[bounds[launch]:bounds[launch + 1]]
    base = r[:, 1].min()
    step = r[:, 0] >> 32
    for s in steps:
        m = step == s
        print(s, [(round((a - base) / 1e3, 1), round((b - base) / 1e3, 1)) for a, b in zip(r[m, 1], r[m, 4])])
