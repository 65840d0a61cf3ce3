#!/usr/bin/env python3
"""Benchmark: slices/s and s/amplitude of the sliced single-amplitude contraction.

A step = one full amplitude: all 2^k ket slices of the workload contracted with the
workload's plan and reduced to one complex128 (sharded over ranks for --gpus N).

Default workload (cfg5bt): BASELINE config 5, the 120-qubit QAOA instance the north-star
target is quoted on (N=120, k=20, 2^20 slices), through the cut and order of
tools/cut_search.cpp under the engine's batched-traffic objective (per-slice peak rank 12;
the reference GA cut + make_job plan peaks at 30 and needs ~1100 s per amplitude on one
B200). Every other config (reference plans, searched orders, searched cuts) is one
--config away.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5bt|cfg5cs|cfg2|cfg1|...]
  python bench.py --impl reference ...    # the reference's CPU path on the same workload

Metric: "slices/s" = 2^k / (seconds per amplitude) (BASELINE.md §3 "ket-equivalent
slices/s"); s_per_amplitude is reported beside it. Timing: CUDA events on the engine's
stream around each pass, barrier + synchronize around the timed region, max over ranks.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")

CONFIGS = {
    "cfg2": dict(stem="cfg2_n60_p1_s1_m10_ext", bitstrings=1,
                 workload="BASELINE config 2: QAOA p=1, seeded 3-regular N=60 (seed 1), k=10 cut edges "
                          "(1024 slices), reference GA (N=40,T=20) + make_job plan, peak rank 16"),
    "cfg1": dict(stem="cfg1_n20_p1_s1_m4", bitstrings=1,
                 workload="BASELINE config 1: QAOA p=1, N=20 (seed 1), k=4 (16 slices), peak rank 7"),
    "cfg4": dict(stem="cfg4_n100_p1_s1_m16_ext", bitstrings=8,
                 workload="BASELINE config 4: QAOA p=1, N=100 (seed 1), k=16 (65536 slices), 8 bitstrings, "
                          "peak rank 22"),
    "cfg5": dict(stem="cfg5_n120_p1_s5_m20_ext", bitstrings=1, sample_passes=4,
                 workload="BASELINE config 5: QAOA p=1, N=120 (seed 5), k=20 (1048576 slices), peak rank 30; "
                          "timed on a sample of whole device passes (all slices are structurally identical), "
                          "s_per_amplitude extrapolated = 2^20 / slices_per_s"),
    # same network and cut, plan from a searched elimination order fed through
    # the reference's own plan_from_order (tools/order_search.cpp, tests/golden/*_os.ref.json)
    "cfg2os": dict(stem="cfg2_n60_p1_s1_m10_ext_os", bitstrings=1,
                   workload="BASELINE config 2 network and cut; order_search plan (peak rank 11, "
                            "reference make_job plan: 16)"),
    "cfg4os": dict(stem="cfg4_n100_p1_s1_m16_ext_os", bitstrings=8,
                   workload="BASELINE config 4 network and cut, 8 bitstrings; order_search plan (peak rank 18, "
                            "reference make_job plan: 22)"),
    "cfg5os": dict(stem="cfg5_n120_p1_s5_m20_ext_os", bitstrings=1, sample_passes=16,
                   workload="BASELINE config 5 network and cut; order_search plan (peak rank 20, reference "
                            "make_job plan: 30); timed on a sample of whole device passes unless --slices "
                            "covers all 2^20 slices"),
    # SURVEY §8(f)-1 extended to the cut: same network and number of cut edges, cut AND order
    # from tools/cut_search.cpp (planned peak of the reference's own plan_from_order on the
    # cut network; tests/golden/*_cs.ref.json). Peaks this low let the reference's own CPU
    # path run the same cut and plan (the reference arm's kind "reference").
    "cfg2cs": dict(stem="cfg2_n60_p1_s1_m10_ext_cs", bitstrings=1,
                   workload="BASELINE config 2 network (N=60, k=10); cut_search cut + order (peak rank 8, "
                            "reference GA cut + make_job plan: 16)"),
    "cfg3cs": dict(stem="cfg3_n50_p2_s1_m14_cs", bitstrings=1,
                   workload="BASELINE config 3: QAOA p=2, seeded 3-regular N=50 (seed 1), k=14 cut edges "
                            "(16384 slices); cut_search cut + order (peak rank 20; the reference GA cut + "
                            "make_job plan peaks at 50, infeasible)"),
    "cfg4cs": dict(stem="cfg4_n100_p1_s1_m16_ext_cs", bitstrings=8,
                   workload="BASELINE config 4 network (N=100, k=16), 8 bitstrings; cut_search cut + order "
                            "(peak rank 9, reference: 22)"),
    "cfg5cs": dict(stem="cfg5_n120_p1_s5_m20_ext_cs", bitstrings=1,
                   workload="BASELINE config 5 network (N=120, k=20, 1048576 slices); cut_search cut + order "
                            "(peak rank 12, reference: 30); every slice of the amplitude per step"),
    "cfg5bt": dict(stem="cfg5_n120_p1_s5_m20_ext_bt", bitstrings=1,
                   workload="BASELINE config 5: QAOA p=1, seeded 3-regular N=120 (seed 5), k=20 cut edges "
                            "(1048576 slices); cut + order from tools/cut_search.cpp with the engine's batched-"
                            "traffic objective, per-slice peak rank 12 (<= 26; the reference GA cut + make_job "
                            "plan: 30); every slice of the amplitude per step"),
    "cfg5bt8": dict(stem="cfg5_n120_p1_s5_m20_ext_bt", bitstrings=8,
                    workload="BASELINE config 5's network, cut and plan (cfg5bt) with 8 output bitstrings "
                             "(SURVEY 8(d) bitstrings 0-7) batched in one pass: 8 x 1048576 slices per step"),
    "cfg2bt": dict(stem="cfg2_n60_p1_s1_m10_ext_bt", bitstrings=1,
                   workload="BASELINE config 2 network (N=60, k=10); cut_search batched-traffic cut + order "
                            "(per-slice peak rank 12; reference GA cut + make_job plan: 16)"),
    "cfg3bt": dict(stem="cfg3_n50_p2_s1_m14_bt", bitstrings=1,
                   workload="BASELINE config 3: QAOA p=2, seeded 3-regular N=50 (seed 1), k=14 cut edges "
                            "(16384 slices); cut_search batched-traffic cut + order (per-slice peak rank 24; the "
                            "reference GA cut + make_job plan peaks at 50, infeasible)"),
    "cfg4bt": dict(stem="cfg4_n100_p1_s1_m16_ext_bt", bitstrings=8,
                   workload="BASELINE config 4 network (N=100, k=16), 8 bitstrings; cut_search batched-traffic "
                            "cut + order (per-slice peak rank 12, reference: 22)"),
}


def instance_info(stem):
    """Generator record of a golden instance (an *_os payload shares its source's)."""
    rec = json.load(open(os.path.join(GOLD, stem + ".ref.json")))
    if "source" in rec:
        rec = json.load(open(os.path.join(GOLD, rec["source"] + ".ref.json")))
    return rec["info"]


def plan_peak(stem):
    import gzip

    with gzip.open(payload(stem), "rt") as f:
        return json.load(f)["plan"]["peak_rank"]


def payload(stem, b=0):
    return os.path.join(GOLD, f"{stem}.b{b}.payload.json.gz")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


class L2Flush:
    """Writes a buffer 4x the B200's 126 MB L2 on the bench device (then synchronizes)."""

    def __init__(self, device):
        import torch

        self.buf = torch.empty(64 << 20, dtype=torch.float64, device=f"cuda:{device}")
        self.device = device

    def __call__(self):
        import torch

        self.buf.fill_(1.0)
        torch.cuda.synchronize(self.device)


def fp64_peak():
    """DFMA peak measured on this pool's B200 by tools/fp64_peak.cu (profiles/r01_fp64_peaks.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")) as f:
            return json.load(f)["dfma_tflops"], "measured (tools/fp64_peak.cu)"
    except Exception:
        return 37.0, "datasheet"


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # QCUT_BENCH_DEVICE pins every rank to one device (several ranks on one GPU: tests only)
    local = int(os.environ.get("QCUT_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        backend = os.environ.get("QCUT_DIST_BACKEND", "nccl")  # gloo: several ranks on one GPU (tests)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def allmax(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch
        import torch.distributed as dist

        dist.barrier()
        torch.cuda.synchronize()


def cpu_port_rate(stem, budget_s=10.0, threads=None):
    """Oracle port (ket view, qcut_oracle.c) over a bounded slice sample on all host threads."""
    from oracle import oracle as O

    threads = threads or os.cpu_count()
    net = O.OracleNet(O.load_payload(payload(stem)), "ket")
    total = net.jobs
    n = min(total, max(threads, 8))
    t0 = time.perf_counter()
    net.sum_range_pool(0, n, threads)
    dt = time.perf_counter() - t0
    per = dt / n
    n2 = int(min(total * 4, max(n, budget_s / max(per, 1e-9))))
    reps, rem = divmod(n2, total)
    t0 = time.perf_counter()
    done = 0
    for _ in range(reps):
        net.sum_range_pool(0, total, threads)
        done += total
    if rem:
        net.sum_range_pool(0, rem, threads)
        done += rem
    dt = time.perf_counter() - t0
    return done / dt, threads, f"ket-view oracle port (qcut_oracle.c), {done} slices of the {total}-slice workload"


def cpu_reference_rate(stem, budget_s=10.0):
    """The compiled reference (oracle/_ref/qcut_refgen bench -> qcut::sum_range on run_pool's grid),
    density view; returns ket-equivalent slices/s = 2^k / (s per amplitude). Whole amplitudes
    when one fits the budget, else the first n density slices (all structurally identical,
    SURVEY §8(d)) and s/amplitude = 4^k / n x their time."""
    refgen = os.path.join(ROOT, "oracle", "_ref", "qcut_refgen")
    import gzip

    tmp = tempfile.NamedTemporaryFile(suffix=".json", delete=False)
    with gzip.open(payload(stem), "rb") as f:
        tmp.write(f.read())
    tmp.close()
    M = instance_info(stem)["M"]
    jobs = 4 ** M
    threads = os.cpu_count()

    def run(n, reps):
        out = subprocess.run([refgen, "bench", "--payload", tmp.name, "--slices", str(n), "--workers",
                              str(threads), "--reps", str(reps)], check=True, capture_output=True, text=True).stdout
        return json.loads(out.strip().splitlines()[-1])["secs"]

    probe = min(jobs, threads)
    t_probe = run(probe, 1)[0]
    est_full = t_probe * jobs / probe
    if est_full <= budget_s:
        secs = run(jobs, max(1, min(50, int(budget_s / max(est_full, 1e-6)))))
        s_amp = statistics.median(secs)
        measured = sum(secs)
        sample = f"reference run_pool grid, {len(secs)} full amplitudes ({jobs} density slices each)"
    else:
        n = min(jobs, probe * max(1, int(budget_s / max(t_probe, 1e-6))))
        measured = run(n, 1)[0]
        s_amp = measured * jobs / n
        sample = (f"reference run_pool grid on the first {n} of {jobs} density slices ({measured:.3g} s measured), "
                  f"s/amplitude extrapolated x{jobs / n:.4g}")
    os.unlink(tmp.name)
    cpu_reference_rate.last_measured_s = measured + t_probe
    return (2 ** M) / s_amp, threads, sample


def reference_arm(args, cfg, world, rank):
    if rank != 0:
        return
    M = instance_info(cfg["stem"])["M"]
    peak = plan_peak(cfg["stem"])
    if peak <= 12:  # 16 * 4^12 B = 268 MB per density tensor: the reference itself runs
        kind = "reference"
        fn = lambda: cpu_reference_rate(cfg["stem"], budget_s=3.0)  # noqa: E731
    else:
        kind = "port"  # reference density view infeasible: 16 * 4^peak B per tensor
        fn = lambda: cpu_port_rate(cfg["stem"], budget_s=3.0)  # noqa: E731
    for _ in range(args.warmup if kind == "port" else 0):
        pass
    rates = []
    sample = ""
    cores = 1
    wall = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r, cores, sample = fn()
        wall.append(time.perf_counter() - t0)
        rates.append(r)
    v = statistics.median(rates)
    line = {
        "impl": "reference", "metric": "slices/s", "value": v, "unit": "slices/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        # a step here is the bounded sample that was really timed; the amplitude time behind
        # `value` (ket-equivalent slices/s = 2^k / s per amplitude) is extrapolated from it
        "ms_per_step": 1e3 * statistics.median(wall), "ms_per_step_is": "wall time of one bounded sample",
        "s_per_amplitude": (2 ** M) / v, "s_per_amplitude_is": "extrapolated from the sample (see cpu_baseline.sample)",
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "complex128", "data": "synthetic (seeded instance from the reference generator)",
        "config": {"workload": cfg["workload"], "k": M, "peak_rank": peak},
        "cpu_baseline": {"value": v, "unit": "slices/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": "slices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if kind == "reference" and peak <= 24:
        # the like-for-like CPU number: the ket-view restatement (the engine's own formulation,
        # no cross-slice sharing) on the same host threads, a bounded sample of the same workload
        pr, pc, ps = cpu_port_rate(cfg["stem"], budget_s=3.0)
        line["like_for_like_port"] = {"value": pr, "unit": "slices/s", "cores": pc, "kind": "port", "sample": ps}
    if kind == "port":
        line["note"] = (f"reference density view infeasible at peak rank {peak} "
                        f"({16 * 4 ** peak:.3g} B per tensor); timed the oracle port in the ket view")
    print(json.dumps(line), flush=True)


def engine_arm(args, cfg, world, rank, local):
    from paper_2010_14962_b200 import Engine
    from paper_2010_14962_b200.shard import aggregate, gather_partials, shard_range

    M = instance_info(cfg["stem"])["M"]
    nb = cfg["bitstrings"]
    amp_shard = args.shard == "amplitudes" and world > 1
    if amp_shard:
        # amplitude-parallel (weak scaling): rank r computes whole amplitudes of its own
        # bitstrings (every slice, no data-path collective); the instance's bitstrings
        # (payloads <stem>.b<i>) are dealt round-robin
        avail = sum(1 for i in range(64) if os.path.exists(payload(cfg["stem"], i)))
        mine = [(rank + world * j) % avail for j in range(nb)]
        pays = [payload(cfg["stem"], b) for b in mine]
    else:
        # several bitstrings share one cut and plan: one engine whose passes carry
        # every amplitude (qc_engine_create_batch), one step = all nb amplitudes
        pays = [payload(cfg["stem"], b) for b in range(nb)]
    engines = [Engine(pays if nb > 1 else pays[0], device=local, mode="ket")]
    st = engines[0].plan_stats()
    if nb > 1 and st["chunks"] > 1:
        # the workspace, not latency, bounds this plan: amplitude bits would only displace slice
        # bits of the pass (measured on config 4's reference plan: 0.229 s per amplitude batched
        # against 0.186 s one amplitude at a time), so every bitstring gets its own engine
        engines[0].close()
        engines = [Engine(p, device=local, mode="ket") for p in pays]
        st = engines[0].plan_stats()
    batched = nb > 1 and len(engines) == 1
    amplitude_slices = 2 ** M
    total = amplitude_slices  # slices per step (whole job)
    if args.slices:
        total = min(total, args.slices * (1 if amp_shard else world))
    elif cfg.get("sample_passes"):
        total = min(total, cfg["sample_passes"] * (2 ** st["batch_bits"]) * (1 if amp_shard else world))
    lo, hi = (0, total) if amp_shard else shard_range(total, rank, world)
    if hi - lo < 2 ** st["batch_bits"]:
        # a rank's shard is smaller than one device pass: cap the batch at the shard so a
        # pass does not compute (and mask) slices of other ranks
        cap = max(0, (hi - lo).bit_length() - 1)
        for e in engines:
            e.close()
        if batched:
            engines = [Engine(pays, device=local, mode="ket", max_batch_bits=cap)]
        else:
            engines = [Engine(p, device=local, mode="ket", max_batch_bits=cap) for p in pays]
        st = engines[0].plan_stats()
    flush = L2Flush(local)
    # cold L2 per timed step: a 512 MB device write in front of it -- unless the pass's working
    # set is itself several times the 126 MB L2 (then every step streams it from HBM anyway)
    big_ws = st["arena_bytes"] > (1 << 30)
    flush_bytes = 0 if big_ws else 512 << 20
    for e in engines:  # warm-up
        e.bench(max(1, args.warmup), lo, hi)
    barrier(world)
    with ClockSampler(local) as clk:
        barrier(world)
        t_dev = 0.0
        res = []
        for _ in range(args.steps):
            # every timed step starts with a cold L2 (a 512 MB device write enqueued on the engine
            # stream in front of the step, outside its CUDA-event bracket): the searched plans'
            # working sets fit the 126 MB L2
            for e in engines:
                r = e.bench_cold(1, lo, hi, flush_bytes=flush_bytes)
                t_dev += sum(r["pass_ms"])
                res.append(r)
        barrier(world)
    clocks = clk.summary()
    launches = engines[0].last_run()["launches"]
    t_max = allmax(t_dev, world)  # ms for K steps (x nb bitstrings)
    amps = args.steps * nb * (world if amp_shard else 1)  # amplitudes of the whole job
    value = total * amps / (t_max / 1e3)  # slices per second, whole job
    s_per_amp = amplitude_slices / value
    # dominant kernel: one instrumented pass (CUDA events around every launch on the
    # engine stream); the launch with the largest share of the pass is reported
    # against the roofline its algorithmic bytes/flops make binding
    prof = engines[0].profile_pass(lo, min(hi, lo + (2 ** st["batch_bits"])))
    dom = max(prof, key=lambda x: x["ms"])
    pass_ms = sum(x["ms"] for x in prof)
    hbm, src = peaks()
    f64, f64src = fp64_peak()
    gbs = dom["bytes"] / (dom["ms"] / 1e3) / 1e9 if dom["ms"] > 0 else 0.0
    # flops the kernel had to execute: the plan's dense count minus what the reference's own
    # zero-skip (contraction.cpp:107-108) removes -- counted by the fused pair kernel
    tfs = dom["exec_flops"] / (dom["ms"] / 1e3) / 1e12 if dom["ms"] > 0 else 0.0
    dense_tfs = dom["flops"] / (dom["ms"] / 1e3) / 1e12 if dom["ms"] > 0 else 0.0
    if gbs / hbm >= tfs / f64:
        roof = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                "peak_source": src}
    else:
        roof = {"bound": "fp64", "achieved": tfs, "peak": f64, "unit": "TFLOP/s", "frac": tfs / f64,
                "peak_source": f64src}
    traffic = None
    try:
        tr = None
        for name in ("r02_traffic.json", "r01_traffic.json"):  # the newest capture that lists this config
            path = os.path.join(ROOT, "profiles", name)
            if tr is None and os.path.exists(path):
                tr = json.load(open(path)).get(args.config)
        if tr and dom["kind"] in tr.get("by_kernel", {}):
            traffic = tr["by_kernel"][dom["kind"]]
        elif tr and tr["kernel"] == dom["kind"]:
            traffic = tr["traffic"]
    except Exception:
        pass
    # the launch that moves the most bytes (the pass's bandwidth-defining kernel; differs from
    # the time-dominant one when the pass is latency-bound)
    big = max(prof, key=lambda x: x["bytes"])
    big_gbs = big["bytes"] / (big["ms"] / 1e3) / 1e9 if big["ms"] > 0 else 0.0
    roof["largest_traffic_launch"] = {"kernel": big["kind"], "ms": big["ms"], "bytes": big["bytes"],
                                      "achieved_gbs": big_gbs, "hbm_frac": big_gbs / hbm,
                                      "share_of_pass": big["ms"] / pass_ms if pass_ms else None}
    if roof["frac"] < 0.1:
        roof["note"] = ("the time-dominant launch is latency-bound (a subtree of dependent small steps: "
                        "k_forest phases / k_flow dataflow levels); the pass moves little data -- see "
                        "largest_traffic_launch and pass_roofline")
    roof.update({"traffic": traffic, "kernel": dom["kind"], "dominant_ms": dom["ms"], "dominant_bytes": dom["bytes"],
                 "dominant_flops": dom["exec_flops"], "dominant_dense_flops": dom["flops"],
                 "hbm_frac": gbs / hbm, "fp64_frac": tfs / f64, "dense_fp64_frac": dense_tfs / f64,
                 "share_of_pass": dom["ms"] / pass_ms if pass_ms else None})
    # e2e through the public API: host pinned upload of the network + result readback per step
    barrier(world)
    t_e2e_local = 0.0
    h2d = d2h = 0
    for _ in range(args.steps):
        for e in engines:
            flush()  # cold L2 per step, outside the timed region
            t0 = time.perf_counter()
            if batched:
                parts = list(e.ket_sum_batch(lo, hi))
            else:
                parts = [e.ket_sum(lo, hi)]
            if world > 1 and not amp_shard:
                # slice shards: one all-gather of (lo, hi, re, im) per amplitude, ordered fold
                sharded = [aggregate(gather_partials(part, lo, hi), total) for part in parts]
            t_e2e_local += time.perf_counter() - t0
            lr = e.last_run()
            h2d += lr["h2d_bytes"]
            d2h += lr["d2h_bytes"]
    t_e2e = allmax(t_e2e_local, world)
    e2e_value = total * amps / t_e2e
    if world > 1 and not amp_shard and len(engines) == 1:
        pass_values = sharded  # the last e2e step's aggregated amplitudes
    elif batched:
        pass_values = list(engines[0].ket_sum_batch(0, total))
    elif world > 1 and not amp_shard:
        pass_values = [aggregate(gather_partials(e.ket_sum(lo, hi), lo, hi), total) for e in engines]
    else:
        pass_values = [e.ket_sum(0, total) for e in engines]
    pass_value = pass_values[0]
    if os.environ.get("QCUT_BENCH_PARTIALS"):  # test hook: this rank's shard and partials
        with open(f"{os.environ['QCUT_BENCH_PARTIALS']}.rank{rank}.json", "w") as f:
            json.dump({"lo": lo, "hi": hi, "batch_bits": st["batch_bits"], "world": world,
                       "partials": [[v.real, v.imag] for v in
                                    (list(engines[0].ket_sum_batch(lo, hi)) if batched
                                     else [e.ket_sum(lo, hi) for e in engines])],
                       "amplitudes": [[v.real, v.imag] for v in pass_values]}, f)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        if st["peak_rank"] > 24:
            cpu = {"value": None, "unit": "slices/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"not run: one ket slice needs 3 x 16 x 2^{st['peak_rank']} B of host RAM"}
        else:
            rate, cores, sample = cpu_port_rate(cfg["stem"], budget_s=args.cpu_seconds)
            cpu = {"value": rate, "unit": "slices/s", "cores": cores, "kind": "port", "sample": sample}
    # algorithmic bytes / flops per amplitude (all passes); a batch engine's plan covers all
    # of its amplitudes at once
    moved_pass = st["moved_bytes"] / max(1, st["n_amplitudes"])
    flops_amp = st["algo_flops"] / max(1, st["n_amplitudes"])
    t_amp = t_max / 1e3 / amps * (amplitude_slices / total)  # s per amplitude (whole job)
    pass_roof = {"algorithmic_bytes_per_amplitude": moved_pass, "algorithmic_flops_per_amplitude": flops_amp,
                 "achieved_gbs": moved_pass / t_amp / 1e9 / world,
                 "achieved_tflops": flops_amp / t_amp / 1e12 / world,
                 "hbm_peak_gbs": hbm, "fp64_peak_tflops": f64,
                 "hbm_frac": moved_pass / t_amp / 1e9 / world / hbm,
                 "fp64_frac": flops_amp / t_amp / 1e12 / world / f64,
                 "note": "per GPU; launches on the pass's critical path run back to back, so a latency-bound "
                         "pass sits far below both rooflines"}
    line = {
        "metric": "slices/s", "value": value, "unit": "slices/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "s_per_amplitude": s_per_amp,
        "higher_is_better": True, "scaling": "weak" if amp_shard else "strong", "vs_baseline": None,
        "dtype": "complex128", "data": "synthetic (seeded instance from the reference generator)",
        "config": {"workload": cfg["workload"], "k": M, "slices_per_amplitude": amplitude_slices,
                   "slices_per_step": total,
                   "amplitudes_per_step": nb, "amplitudes_per_pass": st["n_amplitudes"],
                   "peak_rank": st["peak_rank"], "view": "ket",
                   "batch_bits": st["batch_bits"], "passes": st["chunks"], "arena_bytes": st["arena_bytes"],
                   "l2": (f"working set {st['arena_bytes'] / 1e9:.3g} GB per pass, many times the 126 MB L2 (no flush needed)"
                          if big_ws else
                          f"L2 flushed before every timed step (512 MB device write on the engine stream, outside "
                          f"the event bracket); working set {st['arena_bytes'] / 1e9:.3g} GB"),
                   "sharding": (f"amplitude-parallel: {world} rank(s), each its own bitstring(s) over every slice, "
                                f"no data-path collective" if amp_shard else
                                f"contiguous ket-slice ranges, {world} rank(s), one all-gather of 32 B/rank")},
        "roofline": roof,
        # the whole pass against the same rooflines: the plan's algorithmic bytes (every tensor
        # the engine materialises in HBM -- the batched initial tensors, each launch's inputs
        # and outputs -- read once and written once; intermediates fused into registers or
        # shared memory excluded) and its flops (8 per complex MAC of every plan step at the
        # batched shapes), both per amplitude, over the measured time per amplitude
        "pass_roofline": pass_roof,
        # SURVEY §8(d)'s per-slice count (every step's operands and result per slice, no
        # sharing across slices): a description of the reference's per-slice work, not a
        # throughput denominator -- the engine computes each step once per distinct
        # assignment of the cut bits it depends on
        "s8d_unshared_bytes_per_amplitude": st["essential_bytes"],
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": "slices/s", "h2d_bytes_per_step": h2d // max(1, args.steps),
                "d2h_bytes_per_step": d2h // max(1, args.steps)},
        "gpu_launches": int(launches) * args.steps * nb * world,
        "cpu_baseline": cpu,
        "amplitude": {"re": pass_value.real, "im": pass_value.imag, "abs2": abs(pass_value) ** 2,
                      "note": "ket view, one global phase convention"},
        "amplitudes": [[v.real, v.imag] for v in pass_values] if nb > 1 else None,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    for e in engines:
        e.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", default="cfg5bt", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--shard", default="slices", choices=["slices", "amplitudes"],
                    help="N>1: split one amplitude's slices over the ranks (strong scaling, the default) or give "
                         "every rank whole amplitudes of its own bitstrings (weak scaling)")
    ap.add_argument("--slices", type=int, default=0, help="ket slices per rank per step (default: all, or a "
                    "sample of whole passes for cfg5)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        reference_arm(args, cfg, world, rank)
        return
    world, rank, local = dist_setup(args.gpus)
    engine_arm(args, cfg, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
