#!/usr/bin/env python3
"""BM_ContractPair on the device: the reference's contract_pair microbenchmark
(proj/benchmarks/bench_main.cpp:42-65, shapes (rank, shared) = (4,2) (6,3) (8,4) (9,4)) plus
larger dense shapes, every device path, with the FP64 roofline per shape.

Per shape and path: kernel time (CUDA events on the launch stream, operands resident, mean
of --reps after --warmup), flops = 8 * 4^(2 rank - shared) (the reference's own count), the
fraction of the measured FP64 peaks (profiles/r01_fp64_peaks.json: DFMA 36.35, DMMA 37.10
TFLOP/s) and end-to-end time with host buffers. --cpu also times the UNMODIFIED reference's
contract_pair on this box (oracle/_ref/qcut_refgen pair), one thread as in the reference's
benchmark. One JSON line per shape; --out writes them to a file as a list.
"""
import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2010_14962_b200 import contract_pair_bench  # noqa: E402

PEAK = {"dmma": 37.10, "dfma": 36.35, "small": 36.35}  # TFLOP/s, profiles/r01_fp64_peaks.json
REFGEN = os.path.join(ROOT, "oracle", "_ref", "qcut_refgen")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4:2,6:3,8:4,9:4,10:5,10:4,11:5")
    ap.add_argument("--dim", type=int, default=4)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--paths", default="dmma,dfma,small")
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for spec in args.shapes.split(","):
        rank, k = map(int, spec.split(":"))
        rng = np.random.default_rng(rank * 10 + k)
        n = args.dim ** rank
        a = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        b = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        la = list(range(rank - k, rank))
        lb = list(range(k))
        row = {"rank": rank, "shared": k, "dim": args.dim, "M": args.dim ** (rank - k), "N": args.dim ** (rank - k),
               "K": args.dim ** k, "flops": 8.0 * args.dim ** (2 * rank - k), "paths": {}}
        ref_out = None
        for path in args.paths.split(","):
            if path in ("dmma", "dfma") and row["K"] < 8:
                continue
            if path == "small" and row["flops"] > 3e10:
                continue  # the thin-shape kernel is not meant for these
            reps = args.reps if row["flops"] < 1e11 else max(3, args.reps // 4)
            r = contract_pair_bench(a, la, b, lb, dim=args.dim, path=path, reps=reps, warmup=args.warmup)
            tf = row["flops"] / (r["kernel_ms"] * 1e-3) / 1e12
            row["paths"][path] = {"kernel_ms": r["kernel_ms"], "tflops": tf, "peak_tflops": PEAK[path],
                                  "frac": tf / PEAK[path], "e2e_ms": r["e2e_ms"]}
            if ref_out is None:
                ref_out = r["out"]
            else:
                row["paths"][path]["max_rel_diff_vs_first"] = float(
                    np.max(np.abs(r["out"] - ref_out)) / np.max(np.abs(ref_out)))
        if args.cpu and os.path.exists(REFGEN) and row["flops"] <= 3e9:
            fin = f"/tmp/pair_bench_{rank}_{k}.in"
            with open(fin, "wb") as f:
                f.write(a.tobytes())
                f.write(b.tobytes())
            out = subprocess.run([REFGEN, "pair", "--rank-a", str(rank), "--rank-b", str(rank), "--legs-a",
                                  ",".join(map(str, la)), "--legs-b", ",".join(map(str, lb)), "--in", fin, "--out",
                                  fin + ".out", "--reps", "3"], check=True, capture_output=True, text=True).stdout
            secs = json.loads(out.strip().splitlines()[-1])["secs"]
            got = np.fromfile(fin + ".out", dtype=np.complex128)
            row["cpu_reference"] = {"ms": 1e3 * min(secs), "gflops": row["flops"] / min(secs) / 1e9, "cores": 1,
                                    "kind": "reference",
                                    "max_rel_diff_gpu": float(np.max(np.abs(got - ref_out)) / np.max(np.abs(got)))}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
