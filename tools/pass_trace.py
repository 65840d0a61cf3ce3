#!/usr/bin/env python3
"""Summarise a k_pass item trace (QCG_PASS_TRACE=<file>): per op its kind, tiles, when its first
tile became ready and its last finished, busy time, and the timeline's idle SM time.
    QCG_PASS_TRACE=/tmp/t.bin python tools/time_payload.py <payload>; python tools/pass_trace.py /tmp/t.bin"""
import struct
import sys

import numpy as np

KINDS = ["prep", "forest", "tile", "gate", "gate2", "pair", "chain", "final"]
buf = open(sys.argv[1], "rb").read()
recs = []
at = 0
while at < len(buf):
    n, nops = struct.unpack_from("<QQ", buf, at)
    at += 16
    ops = []
    for i in range(nops):
        kind, desc, var, gx, gy, doff, nd, _pad, item0 = struct.unpack_from("<iiiiiiiiQ", buf, at)
        ops.append(dict(kind=KINDS[kind], gx=gx, gy=gy, ndeps=nd, item0=item0))
        at += 40
    tr = np.frombuffer(buf, dtype=np.uint64, count=4 * n, offset=at).reshape(n, 4)
    at += 32 * n
    recs.append((ops, tr))
ops, tr = recs[-1]
t0 = tr[:, 1].min()
opid = (tr[:, 0] >> 32).astype(int)
sm = (tr[:, 0] & 0xffffffff).astype(int)
claim, ready, done = [(tr[:, k] - t0) / 1e3 for k in (1, 2, 3)]
print(f"pass {done.max():.1f} us, {len(tr)} items, {len(ops)} ops, SMs used {len(set(sm))}")
print(f"sum(done-ready) {np.sum(done - ready):.1f} us  sum(ready-claim) {np.sum(ready - claim):.1f} us")
rows = []
for i, o in enumerate(ops):
    m = opid == i
    if not m.any():
        continue
    rows.append((ready[m].min(), done[m].max(), i, o["kind"], int(m.sum()), np.mean(done[m] - ready[m]),
                 np.max(done[m] - ready[m]), np.mean(ready[m] - claim[m]), o["ndeps"]))
rows.sort()
print(f"{'op':>4} {'kind':7} {'tiles':>6} {'first_ready':>11} {'last_done':>10} {'span':>7} {'mean_tile':>9} {'max_tile':>8} {'mean_wait':>9} deps")
for r in rows:
    print(f"{r[2]:4d} {r[3]:7s} {r[4]:6d} {r[0]:11.1f} {r[1]:10.1f} {r[1]-r[0]:7.1f} {r[5]:9.2f} {r[6]:8.2f} {r[7]:9.2f} {r[8]}")
