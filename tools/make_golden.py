#!/usr/bin/env python3
"""Regenerate tests/golden/ from the UNMODIFIED reference (oracle/_ref/qcut_refgen).

Needs /root/reference (only present in the build container). Every payload and
reference value under tests/golden/ comes from this script; tests never touch
/root/reference at run time.

Instances (SURVEY.md §8(d) derivation: graph random_regular_graph(N, 3, seed),
angles/bitstrings from mix_seed, GA cut search, make_job(restarts=4, seed=1)):

  cfg1_n20_p1_s1_m4    BASELINE config 1 (CPU-runnable): run_serial + all 256 slices
  readme_n12_s7_m2     proj/README.md:44-73 golden example (gamma .6, beta .4, z=0)
  n24_p1_s1_m5         extra p=1 instance, run_serial + 1024 slices
  n10_p2_s1_m4         p=2 instance (peak 10), run_pool(8) value
  cnot / flip          test_executor.cpp:67-80, test_contraction.cpp:158-168
  random_*             helpers.hpp random_circuit + random cut, run_serial + dm_simulate
  cfg2_*, cfg4_*, cfg5_*  BASELINE configs 2, 4 (8 bitstrings), 5: payloads + plan info
                       (the reference CPU path cannot run them: dim-4 peak >= 16)
  *.b0.circuit, *.cut.json  (cfg1, readme) the reference's circuit / cut files (emit_circuit,
                       dump_cut_json with the graph hash) for the file-input path
  cfg3_n50_p2_s1_m14   plan info only: reference planner peak 50 (infeasible)
  *_cs                 (--cut-search, ~25 min) SURVEY §8(f)-1 extended to the cut: the same
                       network with M cut edges AND the order from oracle/_ref/cut_search
                       (joint search scored by the reference's plan_from_order peak); for cfg1
                       the reference's own run_serial on the searched cut is recorded
  mixed_*              (--mixed) random circuits with mixed inputs and non-projector POVMs
                       (general density mode): run_serial, dm_simulate, every slice
  cfg5_*.b1-7          (--cfg5-bitstrings, ~15 min) config 5's bitstrings 1-7 (GA cut of b0 via
                       refgen --cut-from; headline cut and plan) + their oracle amplitudes
  amplitudes.json      (--amplitudes, ~30 min) oracle ket amplitudes (every slice) of configs 2-5
                       through two cuts each, + cfg5 bt reference density slices (refslices)
  dense_triangle.ref.json  (--dense) the reference's run_serial and per-slice values on the dense
                       three-tensor networks of tools/dense_payload.py (payloads rebuilt from
                       their seeds; a checksum of the tensor data pins the generator)
  pairs.npz            (--pairs) qcut::contract_pair itself (the operator under the plan walk): seeded
                       random operands, the reference's result per case -- shapes of
                       BM_ContractPair (bench_main.cpp:60-64) up to rank 6 plus mixed leg orders
  *_os                 (--order-search, ~25 min) SURVEY §8(f)-1: the same network and cut with
                       the plan of oracle/_ref/order_search (a searched elimination order fed
                       through the reference's own plan_from_order); deterministic per seed
"""
import gzip
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
REFGEN = os.path.join(ROOT, "oracle", "_ref", "qcut_refgen")
ORDER_SEARCH = os.path.join(ROOT, "oracle", "_ref", "order_search")
CUT_SEARCH = os.path.join(ROOT, "oracle", "_ref", "cut_search")
TMP = "/tmp/qcut_golden"


def refgen(*args):
    out = subprocess.run([REFGEN, *map(str, args)], check=True, capture_output=True, text=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def gz(src, name):
    with open(src, "rb") as f, gzip.open(os.path.join(GOLD, name), "wb", compresslevel=9) as g:
        g.write(f.read())


def dump(obj, name):
    with open(os.path.join(GOLD, name), "w") as f:
        json.dump(obj, f, indent=1)
        f.write("\n")


def copy(src, name):
    with open(src, "rb") as f, open(os.path.join(GOLD, name), "wb") as g:
        g.write(f.read())


def qaoa(name, n, p, seed, M, slices=False, pool=False, bitstrings=1, run=True, extra=(), files=False):
    prefix = os.path.join(TMP, name)
    info = refgen("gen", "--n", n, "--p", p, "--seed", seed, "--M", M, "--bitstrings", bitstrings,
                  "--out", prefix, *extra)
    rec = {"info": info}
    for b in range(bitstrings):
        gz(f"{prefix}.b{b}.payload.json", f"{name}.b{b}.payload.json.gz")
    if files:  # the reference's on-disk inputs of `qcut run`
        copy(f"{prefix}.b0.circuit", f"{name}.b0.circuit")
        copy(f"{prefix}.cut.json", f"{name}.cut.json")
    if run:
        pay = f"{prefix}.b0.payload.json"
        if pool:
            r = refgen("bench", "--payload", pay, "--slices", 4 ** M, "--workers", 8)
            rec["run_pool8"] = r["value"]
            rec["pool_secs"] = r["secs"]
        else:
            r = refgen("run", "--payload", pay, "--slices", 1 if slices else 0, "--steps", 1)
            rec["run_serial"] = r["value"]
            rec["serial_secs"] = r["secs"]
            rec["steps"] = r["steps"]
            if slices:
                rec["slices"] = r["slices"]
    dump(rec, f"{name}.ref.json")
    print(name, json.dumps(info.get("plan")), flush=True)


def main():
    if not os.path.exists(REFGEN):
        sys.exit("build oracle/_ref first: make -C oracle ref")
    os.makedirs(GOLD, exist_ok=True)
    os.makedirs(TMP, exist_ok=True)
    qaoa("cfg1_n20_p1_s1_m4", 20, 1, 1, 4, slices=True, files=True)
    qaoa("readme_n12_s7_m2", 12, 1, 7, 2, slices=True, files=True,
         extra=("--ga-seed", 1, "--gamma", 0.6, "--beta", 0.4, "--zeros"))
    qaoa("n24_p1_s1_m5", 24, 1, 1, 5, slices=True)
    qaoa("n10_p2_s1_m4", 10, 2, 1, 4, pool=True)
    for name, flag in (("cnot", ()), ("flip", ("--flip",))):
        path = os.path.join(TMP, name + ".payload.json")
        r = refgen("cnot", "--out", path, *flag)
        gz(path, name + ".payload.json.gz")
        dump({"run_serial": r["serial"]}, name + ".ref.json")
    cases = [(3, 8, 5, 2), (4, 10, 7, 3), (2, 6, 11, 1), (5, 14, 13, 3), (3, 12, 17, 4), (6, 15, 19, 2),
             (1, 5, 23, 1), (4, 9, 29, 2)]
    for n, depth, seed, M in cases:
        name = f"random_n{n}_d{depth}_s{seed}_m{M}"
        path = os.path.join(TMP, name + ".payload.json")
        r = refgen("random", "--n", n, "--depth", depth, "--seed", seed, "--M", M, "--out", path)
        slices = refgen("run", "--payload", path, "--slices", 1)
        r["slices"] = slices["slices"]
        gz(path, name + ".payload.json.gz")
        dump(r, name + ".ref.json")
        print(name, r["serial"], r.get("dm_simulate"), flush=True)
    ext = ("--ga-n", 40, "--ga-t", 20)
    qaoa("cfg2_n60_p1_s1_m10_ext", 60, 1, 1, 10, run=False, extra=ext)
    qaoa("cfg2_n60_p1_s1_m10", 60, 1, 1, 10, run=False)
    qaoa("cfg4_n100_p1_s1_m16_ext", 100, 1, 1, 16, run=False, bitstrings=8, extra=ext)
    qaoa("cfg5_n120_p1_s5_m20_ext", 120, 1, 5, 20, run=False, extra=ext)
    info = refgen("gen", "--n", 50, "--p", 2, "--seed", 1, "--M", 14, "--out", os.path.join(TMP, "cfg3"))
    dump({"info": info, "note": "reference planner peak rank 50: 2^50 x 16 B per tensor, infeasible"},
         "cfg3_n50_p2_s1_m14.ref.json")


def order_search(src, tmp_src, evals, seed, bitstrings=1, split=False):
    """<src>_os payloads: src's network + cut, plan from order_search (same plan for every
    bitstring: plans depend only on structure). split=True: <src>_split, the
    opt-in 2-qubit operator-Schmidt split of the network (order_search --split-2q 1), one
    bitstring; its reference run_serial is recorded when the reference can run it."""
    name = src + ("_split" if split else "_os")
    out = os.path.join(TMP, name + ".b0.payload.json")
    log = out + ".log"
    if not (os.path.exists(out) and os.path.exists(log)):
        r = subprocess.run([ORDER_SEARCH, "--payload", tmp_src(0), "--out", out, "--evals", str(evals),
                            "--seed", str(seed)] + (["--split-2q", "1"] if split else []),
                           check=True, capture_output=True, text=True)
        with open(log, "w") as f:
            f.write(r.stdout)
    res = json.loads(open(log).read().strip().splitlines()[-1])
    plan = json.load(open(out))
    rec = {"source": src, "order_search": res, "evals": evals, "seed": seed,
           "command": f"order_search --payload {src}.b0 --evals {evals} --seed {seed}" +
                      (" --split-2q 1" if split else "")}
    if split:
        gz(out, f"{name}.b0.payload.json.gz")
        if plan["plan"]["peak_rank"] <= 8:
            rec["run_serial"] = refgen("run", "--payload", out, "--slices", 0, "--steps", 0)["value"]
    else:
        for b in range(bitstrings):
            pay = json.load(open(tmp_src(b)))
            pay["plan"], pay["max_rank"] = plan["plan"], plan["max_rank"]
            with gzip.open(os.path.join(GOLD, f"{name}.b{b}.payload.json.gz"), "wt", compresslevel=9) as g:
                json.dump(pay, g, separators=(",", ":"))
    dump(rec, name + ".ref.json")
    print(name, json.dumps(res), flush=True)


def order_searches():
    t = lambda stem: (lambda b: os.path.join(TMP, f"{stem}.b{b}.payload.json"))  # noqa: E731
    order_search("cfg2_n60_p1_s1_m10_ext", t("cfg2_n60_p1_s1_m10_ext"), 20000, 1)
    order_search("cfg4_n100_p1_s1_m16_ext", t("cfg4_n100_p1_s1_m16_ext"), 40000, 1, bitstrings=8)
    order_search("cfg5_n120_p1_s5_m20_ext", t("cfg5_n120_p1_s5_m20_ext"), 80000, 2)
    order_search("cfg3_n50_p2_s1_m14", t("cfg3"), 80000, 3)
    order_search("cfg1_n20_p1_s1_m4", t("cfg1_n20_p1_s1_m4"), 3000, 1, split=True)
    order_search("cfg2_n60_p1_s1_m10_ext", t("cfg2_n60_p1_s1_m10_ext"), 20000, 1, split=True)


def cut_search(name, src, evals, seed, bitstrings=1, run=False, threads=8, ref_range=None, source=None, extra=(),
               rerank=False):
    """<name>: src's network (tests/golden/<src>.b*.payload.json.gz, or a TMP payload path
    for src) with the cut AND plan of cut_search (same M). Cuts and plans depend only on
    structure, so every bitstring's payload gets the same cut and plan.
    run=True records the reference's own run_serial on the searched cut (density view);
    rerank=True keeps, among the 8 chains' results (--emit-all), the one whose plan the
    engine's own host planner moves the fewest bytes for (tools/rerank_plans.py);
    ref_range=(lo, hi) records the reference's per-slice values sum_range(s, s+1) for the
    density slice ids in [lo, hi) and sum_range(lo, hi) (the searched plans are small
    enough for the reference's CPU path even where its own plan is not)."""
    os.makedirs(TMP, exist_ok=True)
    def src_path(b):
        if src.endswith(".json"):
            return src.replace(".b0.", f".b{b}.")
        path = os.path.join(TMP, f"{src}.b{b}.payload.json")
        with gzip.open(os.path.join(GOLD, f"{src}.b{b}.payload.json.gz"), "rb") as f, open(path, "wb") as g:
            g.write(f.read())
        return path
    out = os.path.join(TMP, name + ".b0.payload.json")
    log = out + ".log"
    cmd = ["--payload", src_path(0), "--out", out, "--evals", str(evals), "--seed", str(seed),
           "--threads", str(threads), *map(str, extra)]
    if rerank:
        cmd += ["--emit-all", "1"]
    if not (os.path.exists(out) and os.path.exists(log)):
        r = subprocess.run([CUT_SEARCH, *cmd], check=True, capture_output=True, text=True)
        with open(log, "w") as f:
            f.write(r.stdout)
    res = json.loads(open(log).read().strip().splitlines()[-1])
    chosen = out
    if rerank:
        sys.path.insert(0, ROOT)
        from tools.rerank_plans import engine_cost
        cands = [out] + [f"{out}.t{t}.json" for t in range(threads)]
        costs = {c: engine_cost(c)[0] for c in cands if os.path.exists(c)}
        chosen = min(costs, key=lambda c: (costs[c], c))
        res["rerank"] = {"chosen": os.path.basename(chosen).replace(name + ".b0.payload.json", "<main>"),
                         "engine_moved_bytes": {os.path.basename(c).replace(name + ".b0.payload.json", "<main>"): v
                                                for c, v in costs.items()}}
    plan = json.load(open(chosen))
    out = chosen
    rec = {"source": source or src, "cut_search": res,
           "evals": evals, "seed": seed, "threads": threads,
           "command": f"cut_search --payload <source>.b0 --evals {evals} --seed {seed} --threads {threads}" +
                      "".join(f" {x}" for x in extra)}
    for b in range(bitstrings):
        pay = json.load(open(src_path(b)))
        assert pay["network"]["edges"] == plan["network"]["edges"]
        pay["cut"], pay["plan"], pay["max_rank"] = plan["cut"], plan["plan"], plan["max_rank"]
        with gzip.open(os.path.join(GOLD, f"{name}.b{b}.payload.json.gz"), "wt", compresslevel=9) as g:
            json.dump(pay, g, separators=(",", ":"))
    if run:
        r = refgen("run", "--payload", out, "--slices", 1, "--steps", 0)
        rec["run_serial"], rec["slices"] = r["value"], r["slices"]
    if ref_range and ref_range[0] == "peak":
        # start at the density slice (k, k) of the largest ket slice among the first
        # ref_range[1] (ket oracle), so the recorded reference values are far from zero
        sys.path.insert(0, ROOT)
        from oracle import oracle as O
        import numpy as np
        net = O.OracleNet(O.load_payload(out), "ket")
        _, kv = net.sum_range(0, ref_range[1], per_slice=True)
        k, M = int(np.argmax(np.abs(kv))), len(plan["cut"])
        d = sum(3 << (2 * (M - 1 - i)) if (k >> (M - 1 - i)) & 1 else 0 for i in range(M))
        ref_range = (d, d + ref_range[2])
    if ref_range:
        r = refgen("run", "--payload", out, "--lo", ref_range[0], "--hi", ref_range[1], "--slices", 1)
        rec["ref_range"] = {"lo": ref_range[0], "hi": ref_range[1], "sum_range": r["value"],
                            "slices": r["slices"], "secs": r["secs"]}
    dump(rec, name + ".ref.json")
    print(name, json.dumps(res), flush=True)


def cut_searches():
    cut_search("cfg1_n20_p1_s1_m4_cs", "cfg1_n20_p1_s1_m4", 20000, 1, run=True)
    cut_search("cfg2_n60_p1_s1_m10_ext_cs", "cfg2_n60_p1_s1_m10_ext", 600000, 1, ref_range=(0, 4096))
    cut_search("cfg4_n100_p1_s1_m16_ext_cs", "cfg4_n100_p1_s1_m16_ext", 1000000, 1, bitstrings=8,
               ref_range=("peak", 4096, 64))
    cut_search("cfg5_n120_p1_s5_m20_ext_cs", "cfg5_n120_p1_s5_m20_ext", 1000000, 1, ref_range=("peak", 256, 2))
    # config 3: the reference planner peaks at 50 on the GA cut; two searched cuts (seeds 3, 2)
    # give two independent slicings of one network (cross-cut amplitude identity)
    refgen("gen", "--n", 50, "--p", 2, "--seed", 1, "--M", 14, "--out", os.path.join(TMP, "cfg3"))
    cfg3 = os.path.join(TMP, "cfg3.b0.payload.json")
    cut_search("cfg3_n50_p2_s1_m14_cs", cfg3, 1500000, 3, source="cfg3_n50_p2_s1_m14")
    cut_search("cfg3_n50_p2_s1_m14_cs2", cfg3, 400000, 2, source="cfg3_n50_p2_s1_m14")
    # *_bt: the engine's batched-traffic objective (every slice a batch bit of the tensors
    # that depend on it), per-slice peak bounded so the reference's CPU path still runs a
    # density slice where it can (bound 12)
    bt = ("--objective", "batched", "--cap", 31)
    # (seed 54 at 2M evaluations: of the 20 seeds tried (7, 11-14, 21-22, 31-32, 51-58), the
    # plan with the fewest engine-moved bytes (0.17 GB, tools/rerank_plans.py) and the fastest
    # measured amplitude (tools/time_payload.py: 0.18 ms vs 0.23 ms for seed 11's 0.21 GB))
    cut_search("cfg5_n120_p1_s5_m20_ext_bt", "cfg5_n120_p1_s5_m20_ext", 2000000, 54, ref_range=("peak", 256, 2),
               extra=bt + ("--bound", 12, "--emit-all", 1))
    cut_search("cfg2_n60_p1_s1_m10_ext_bt", "cfg2_n60_p1_s1_m10_ext", 600000, 7, ref_range=("peak", 1024, 64),
               extra=bt + ("--bound", 12))
    cut_search("cfg4_n100_p1_s1_m16_ext_bt", "cfg4_n100_p1_s1_m16_ext", 1000000, 7, bitstrings=8,
               ref_range=("peak", 4096, 16), extra=bt + ("--bound", 12))
    cut_search("cfg3_n50_p2_s1_m14_bt", cfg3, 1000000, 7, source="cfg3_n50_p2_s1_m14", extra=bt + ("--bound", 24))


def ket_slices_threaded(stem, b=0, threads=8):
    """Every ket slice value A(k) of <stem>.b<b> by the C oracle (qcut_oracle.c, ket view),
    contiguous chunks on `threads` Python threads (ctypes releases the GIL)."""
    import threading

    import numpy as np

    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    net = O.OracleNet(O.load_payload(os.path.join(GOLD, f"{stem}.b{b}.payload.json.gz")), "ket")
    n = net.jobs
    out = np.zeros(n, dtype=np.complex128)
    chunk = max(1, (n + 8 * threads - 1) // (8 * threads))
    todo = list(range(0, n, chunk))
    lock = threading.Lock()

    def work():
        while True:
            with lock:
                if not todo:
                    return
                lo = todo.pop(0)
            hi = min(n, lo + chunk)
            _, v = net.sum_range(lo, hi, per_slice=True)
            out[lo:hi] = v

    th = [threading.Thread(target=work) for _ in range(threads)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return out


def amp_record(vals, M):
    """Amplitude-level fixture of one (network, bitstring, plan): A = sum_k A(k) (correctly
    rounded fsum), sum_k |A(k)|^2, a seeded-weight checksum sum_k w_k A(k) with
    w_k = cos(0.7 k) (size-independent projection of all 2^M values), the 64 largest slices
    and 64 strided slices with their ids."""
    import math

    import numpy as np

    k = np.arange(len(vals), dtype=np.float64)
    w = np.cos(0.7 * k)
    top = np.argsort(-np.abs(vals), kind="stable")[:64]
    stride = max(1, len(vals) // 64)
    strided = np.arange(7 % len(vals), len(vals), stride)[:64]
    A = complex(math.fsum(vals.real), math.fsum(vals.imag))
    return {
        "M": M,
        "A": [A.real, A.imag],
        "abs2": abs(A) ** 2,
        "sum_abs2": math.fsum(np.abs(vals) ** 2),
        "checksum_cos07": [math.fsum(w * vals.real), math.fsum(w * vals.imag)],
        "top_ids": [int(i) for i in top],
        "top_vals": [[float(vals[i].real), float(vals[i].imag)] for i in top],
        "strided_ids": [int(i) for i in strided],
        "strided_vals": [[float(vals[i].real), float(vals[i].imag)] for i in strided],
    }


def amplitudes():
    """tests/golden/amplitudes.json: oracle ket amplitudes (every slice, qcut_oracle.c) for the
    headline and configs 2-5, each through two independent cuts where affordable (the amplitude
    is cut-independent: a cut only splits the same contraction, cutting.hpp:41-46, and the ket
    factors, hence the global phase, belong to the network). Plus <cfg5 bt>.refslices.json:
    the compiled reference's own density-slice values sum_range(s, s+1) (executor.cpp:45-68) on
    256 ids d(k, b) for the 16 largest ket slices k, b, and 64 strided ids."""
    import time

    import numpy as np

    todo = [  # (network key, plan stems, bitstrings)
        ("cfg5_n120_p1_s5_m20_ext", ["cfg5_n120_p1_s5_m20_ext_bt", "cfg5_n120_p1_s5_m20_ext_cs"], 1),
        ("cfg4_n100_p1_s1_m16_ext", ["cfg4_n100_p1_s1_m16_ext_bt", "cfg4_n100_p1_s1_m16_ext_cs"], 8),
        ("cfg2_n60_p1_s1_m10_ext", ["cfg2_n60_p1_s1_m10_ext_bt", "cfg2_n60_p1_s1_m10_ext"], 1),
        ("cfg3_n50_p2_s1_m14", ["cfg3_n50_p2_s1_m14_cs"], 1),
    ]
    path = os.path.join(GOLD, "amplitudes.json")
    rec = json.load(open(path)) if os.path.exists(path) else {}
    for net, stems, nb in todo:
        for b in range(nb):
            for stem in stems:
                key = f"{stem}.b{b}"
                if key in rec:
                    continue
                M = len(json.load(gzip.open(os.path.join(GOLD, f"{stem}.b{b}.payload.json.gz"), "rt"))["cut"])
                t0 = time.time()
                vals = ket_slices_threaded(stem, b)
                r = amp_record(vals, M)
                r.update({"network": net, "bitstring": b, "secs": time.time() - t0, "threads": 8,
                          "method": "qcut_oracle.c ket view, every slice, fsum in double"})
                rec[key] = r
                print(key, r["A"], f"{r['secs']:.1f}s", flush=True)
                dump(rec, "amplitudes.json")
                if stem == "cfg5_n120_p1_s5_m20_ext_bt" and b == 0:
                    top = np.argsort(-np.abs(vals), kind="stable")[:16]
                    ids = []
                    for k in top:
                        for bb in top:  # density digit d_i = 2 k_i + b_i, MSB = first cut edge
                            ids.append(sum(((((int(k) >> (M - 1 - i)) & 1) << 1) | ((int(bb) >> (M - 1 - i)) & 1))
                                           << (2 * (M - 1 - i)) for i in range(M)))
                    stride = 4 ** M // 64
                    ids += [12345 + j * stride for j in range(64)]
                    out = os.path.join(TMP, stem + ".b0.payload.json")
                    with gzip.open(os.path.join(GOLD, f"{stem}.b0.payload.json.gz"), "rb") as f, open(out, "wb") as g:
                        g.write(f.read())
                    r2 = refgen("slices", "--payload", out, "--ids", ",".join(map(str, ids)), "--workers", 8)
                    dump({"source": stem, "command": "qcut_refgen slices (qcut::sum_range(job, s, s+1) per id)",
                          "ids": r2["ids"], "slices": r2["slices"], "secs": r2["secs"],
                          "note": "256 ids d(k,b) over the 16 largest ket slices k, b (oracle), then 64 "
                                  "strided ids 12345 + j * 4^M/64"},
                         stem + ".refslices.json")
                    print("refslices", len(ids), f"{r2['secs']:.1f}s", flush=True)
    # cross-plan agreement on the oracle itself (independent cuts of one network)
    for net, stems, nb in todo:
        for b in range(nb):
            vals = [complex(*rec[f"{s}.b{b}"]["A"]) for s in stems if f"{s}.b{b}" in rec]
            if len(vals) > 1:
                d = max(abs(v - vals[0]) for v in vals) / abs(vals[0])
                print(net, b, "cross-cut rel diff", d)
                assert d < 1e-10, (net, b, d)


MIXED_CASES = [(8, 48, 41, 4), (6, 30, 43, 5), (4, 14, 5, 3)]


def mixed():
    """mixed_*: general density mode -- the reference test generator's random
    circuits with mixed inputs and non-projector POVM elements (refgen mixed): run_serial,
    dm_simulate and every per-slice value of the reference. The ket view cannot run them."""
    os.makedirs(TMP, exist_ok=True)
    for n, depth, seed, M in MIXED_CASES:
        name = f"mixed_n{n}_d{depth}_s{seed}_m{M}"
        path = os.path.join(TMP, name + ".payload.json")
        r = refgen("mixed", "--n", n, "--depth", depth, "--seed", seed, "--M", M, "--out", path)
        gz(path, name + ".payload.json.gz")
        dump(r, name + ".ref.json")
        print(name, r["serial"], r.get("dm_simulate"), flush=True)


def cfg5_bitstrings():
    """Bitstrings 1-7 of the config 5 instance (amplitude-parallel multi-GPU bench and batch
    tests): the same network (graph seed 5) with the SURVEY §8(d) bitstrings b = 1..7, the GA
    cut of <ext>.b0 (refgen --cut-from: plans and cuts depend only on structure), and for the
    headline plan the cut and plan of <ext_bt>.b0. Their oracle amplitudes join amplitudes.json."""
    src = "cfg5_n120_p1_s5_m20_ext"
    os.makedirs(TMP, exist_ok=True)
    b0 = os.path.join(TMP, src + ".b0.src.json")
    with gzip.open(os.path.join(GOLD, src + ".b0.payload.json.gz"), "rb") as f, open(b0, "wb") as g:
        g.write(f.read())
    prefix = os.path.join(TMP, "cfg5x")
    refgen("gen", "--n", 120, "--p", 1, "--seed", 5, "--M", 20, "--bitstrings", 8, "--cut-from", b0,
           "--ga-n", 40, "--ga-t", 20, "--out", prefix)
    want = json.load(open(b0))
    got = json.load(open(prefix + ".b0.payload.json"))
    assert got == want, "regenerated bitstring 0 differs from the committed payload"
    bt = json.load(gzip.open(os.path.join(GOLD, src + "_bt.b0.payload.json.gz"), "rt"))
    for b in range(1, 8):
        pay = json.load(open(f"{prefix}.b{b}.payload.json"))
        assert pay["network"]["edges"] == bt["network"]["edges"] and pay["cut"] == want["cut"]
        gz(f"{prefix}.b{b}.payload.json", f"{src}.b{b}.payload.json.gz")
        pay["cut"], pay["plan"], pay["max_rank"] = bt["cut"], bt["plan"], bt["max_rank"]
        with gzip.open(os.path.join(GOLD, f"{src}_bt.b{b}.payload.json.gz"), "wt", compresslevel=9) as g:
            json.dump(pay, g, separators=(",", ":"))
    path = os.path.join(GOLD, "amplitudes.json")
    rec = json.load(open(path))
    import time
    for b in range(1, 8):
        key = f"{src}_bt.b{b}"
        if key in rec:
            continue
        t0 = time.time()
        r = amp_record(ket_slices_threaded(src + "_bt", b), 20)
        r.update({"network": src, "bitstring": b, "secs": time.time() - t0, "threads": 8,
                  "method": "qcut_oracle.c ket view, every slice, fsum in double"})
        rec[key] = r
        dump(rec, "amplitudes.json")
        print(key, r["A"], f"{r['secs']:.1f}s", flush=True)


# (rank_a, legs_a, rank_b, legs_b): BM_ContractPair's layouts (shared legs last in a, first in
# b) and permuted ones (test_contraction.cpp:64-106 exercise leg order on both sides)
PAIR_CASES = [
    (2, [1], 2, [0]), (2, [0], 2, [0]), (4, [2, 3], 4, [0, 1]), (5, [3, 4], 5, [0, 1]),
    (5, [0, 3], 4, [2, 1]), (4, [1], 3, [2]), (6, [3, 4, 5], 6, [0, 1, 2]), (6, [4, 0, 2], 5, [1, 3, 0]),
    (3, [0, 1, 2], 5, [4, 0, 2]), (6, [1, 2, 3, 4], 5, [3, 2, 1, 0]),
]


def pairs():
    """pairs.npz: for every PAIR_CASES entry the operands (numpy default_rng(seed), uniform in
    [-1, 1) like bench_main.cpp's random_tensor) and the reference's contract_pair result."""
    import numpy as np
    os.makedirs(TMP, exist_ok=True)
    rec = {}
    for i, (ra, la, rb, lb) in enumerate(PAIR_CASES):
        rng = np.random.default_rng(1000 + i)
        a = rng.uniform(-1, 1, 4 ** ra) + 1j * rng.uniform(-1, 1, 4 ** ra)
        b = rng.uniform(-1, 1, 4 ** rb) + 1j * rng.uniform(-1, 1, 4 ** rb)
        if i == 3:  # zero entries take the reference's skip branch (contraction.cpp:107-108)
            a[::3] = 0
        fin, fout = os.path.join(TMP, f"pair{i}.in"), os.path.join(TMP, f"pair{i}.out")
        with open(fin, "wb") as f:
            f.write(a.astype(np.complex128).tobytes())
            f.write(b.astype(np.complex128).tobytes())
        r = refgen("pair", "--rank-a", ra, "--rank-b", rb, "--legs-a", ",".join(map(str, la)),
                   "--legs-b", ",".join(map(str, lb)), "--in", fin, "--out", fout)
        out = np.fromfile(fout, dtype=np.complex128)
        assert r["rank"] == ra + rb - 2 * len(la) and out.size == 4 ** r["rank"]
        rec[f"a{i}"], rec[f"b{i}"], rec[f"out{i}"] = a, b, out
        rec[f"spec{i}"] = np.array([ra, rb, len(la)] + la + lb, dtype=np.int32)
        print("pair", i, ra, la, rb, lb, "->", r["rank"], flush=True)
    np.savez_compressed(os.path.join(GOLD, "pairs.npz"), **rec)


DENSE_CASES = [(5, 3, 3, 7), (4, 3, 3, 11), (6, 2, 3, 5)]  # (a, b, c, seed), tools/dense_payload.py


def dense():
    """dense_triangle.ref.json: the reference on the dense networks (one PlanStep is an
    M x K x N = 4^c x 4^(a-1) x 4^b contraction per slice; cut edge 0)."""
    import numpy as np
    sys.path.insert(0, ROOT)
    from tools.dense_payload import dense_triangle, dense_value
    os.makedirs(TMP, exist_ok=True)
    rec = {}
    for a, b, c, seed in DENSE_CASES:
        pay, data = dense_triangle(a, b, c, seed)
        path = os.path.join(TMP, f"dense_{a}_{b}_{c}_{seed}.json")
        with open(path, "w") as f:
            json.dump(pay, f, separators=(",", ":"))
        r = refgen("run", "--payload", path, "--slices", 1, "--steps", 1)
        want = dense_value(a, b, c, data)
        assert abs(complex(*r["value"]) - want) <= 1e-12 * abs(want), (r["value"], want)
        rec[f"{a}_{b}_{c}_{seed}"] = {"run_serial": r["value"], "slices": r["slices"], "steps": r["steps"],
                                      "checksum": float(sum(np.sum(np.abs(d)) for d in data))}
        print("dense", a, b, c, seed, r["value"], flush=True)
    dump(rec, "dense_triangle.ref.json")


if __name__ == "__main__":
    if "--dense" in sys.argv:
        dense()
        sys.exit(0)
    if "--pairs" in sys.argv:
        pairs()
        sys.exit(0)
    if "--mixed" in sys.argv:
        mixed()
        sys.exit(0)
    if "--cfg5-bitstrings" in sys.argv:
        cfg5_bitstrings()
        sys.exit(0)
    if "--amplitudes" in sys.argv:
        os.makedirs(TMP, exist_ok=True)
        amplitudes()
        sys.exit(0)
    if "--cut-search" in sys.argv:
        cut_searches()
        sys.exit(0)
    if "--order-search" in sys.argv:
        order_searches()
        sys.exit(0)
    main()
