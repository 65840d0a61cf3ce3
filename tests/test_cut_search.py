"""SURVEY §8(f)-1 extended to the cut: payloads whose cut edges AND elimination order come
from oracle/_ref/cut_search (tools/cut_search.cpp), a joint search scored by the planned
peak of the reference's own plan_from_order (contraction.cpp:118-262) on the cut network.

A *_cs payload keeps its source's network and the number of cut edges M; the cut set and
the plan change, so slice ids do not correspond across cuts, but the amplitude does: the
sum over all slices of any cut is the same contraction of the same network
(cutting.hpp:41-46, test_cutting.cpp:118-149). Parity is pinned three ways:
  * the reference's OWN executor on the searched cut: run_serial (cfg1) and per-slice
    density values over ranges of the N=60/100/120 instances (make_golden.py records them;
    the searched plans are small enough for the reference's CPU path) — against the oracle
    here and the engine on the GPU;
  * cross-cut identity: |A|^2 over all slices of the searched cut equals |A|^2 of the
    reference's GA cut (cfg1 by the reference itself, cfg2/4/5 on the oracle or engine) and
    of a second searched cut (cfg3, whose GA cut no plan can run: peak >= 35);
  * the ket oracle per slice on the searched plans.
"""
import gzip
import json

import numpy as np
import pytest

from conftest import cx, payload_path, ref_json

REL = 1e-10
CS = {  # cs stem -> (source stem or None, bitstrings, BASELINE rank bound)
    "cfg1_n20_p1_s1_m4_cs": ("cfg1_n20_p1_s1_m4", 1, None),
    "cfg2_n60_p1_s1_m10_ext_cs": ("cfg2_n60_p1_s1_m10_ext", 1, 22),
    "cfg3_n50_p2_s1_m14_cs": (None, 1, 24),
    "cfg3_n50_p2_s1_m14_cs2": (None, 1, 24),
    "cfg4_n100_p1_s1_m16_ext_cs": ("cfg4_n100_p1_s1_m16_ext", 8, 24),
    "cfg5_n120_p1_s5_m20_ext_cs": ("cfg5_n120_p1_s5_m20_ext", 1, 26),
    # batched-traffic objective (the engine's cost model), per-slice peak bounded at 12
    "cfg5_n120_p1_s5_m20_ext_bt": ("cfg5_n120_p1_s5_m20_ext", 1, 12),
    "cfg2_n60_p1_s1_m10_ext_bt": ("cfg2_n60_p1_s1_m10_ext", 1, 12),
    "cfg4_n100_p1_s1_m16_ext_bt": ("cfg4_n100_p1_s1_m16_ext", 8, 12),
    "cfg3_n50_p2_s1_m14_bt": (None, 1, 24),
}


def load(stem, b=0):
    with gzip.open(payload_path(stem, b), "rt") as f:
        return json.load(f)


def maxdiff(a, ref):
    return np.max(np.abs(a - ref)) / np.abs(ref).max()


def dephase(a, ref):
    c = np.vdot(a, ref)
    return a * (c / abs(c)) if abs(c) > 0 else a


@pytest.mark.parametrize("stem", sorted(CS))
def test_cs_payload_keeps_network_and_cut_size(stem):
    src, nb, bound = CS[stem]
    rec = ref_json(stem)["cut_search"]
    for b in range(nb):
        p = load(stem, b)
        assert p["cut"] == sorted(set(p["cut"])) == rec["cut"] and len(p["cut"]) == rec["M"]
        assert len(p["plan"]["steps"]) == rec["steps"] and p["plan"]["peak_rank"] == rec["peak"]
        if src:
            q = load(src, b)
            assert p["network"] == q["network"] and p["v"] == q["v"] and len(p["cut"]) == len(q["cut"])
            assert rec["reference_peak"] == q["plan"]["peak_rank"]
    assert rec["peak"] < rec["reference_peak"]
    if rec.get("objective") == "batched":
        assert "--objective batched" in ref_json(stem)["command"]
    if bound:
        assert rec["peak"] <= bound  # BASELINE.json's per-slice rank bound for the config
    if stem.startswith("cfg3"):
        info = ref_json("cfg3_n50_p2_s1_m14")["info"]
        assert rec["M"] == info["M"] == 14 and rec["reference_peak"] == info["max_rank"] == 50


@pytest.mark.parametrize("stem", sorted(CS))
def test_cs_host_program_valid(stem):
    from paper_2010_14962_b200 import Engine

    with Engine(payload_path(stem), device=-1, mode="ket") as e:
        st = e.plan_stats()
    assert st["peak_rank"] == ref_json(stem)["cut_search"]["peak"]
    assert st["n_cut"] == ref_json(stem)["cut_search"]["M"] and st["ket_jobs"] == 2 ** st["n_cut"]


def test_forest_units_cover_first_group(monkeypatch):
    """Config 5's first dataflow group (617 small steps) runs as k_forest: one CTA per
    independent subtree (35 roots), phases = the deepest subtree's depth; the subtrees are
    split over up to three launches by estimated time (QCG_FOREST_SPLIT=0: one launch). With the forest
    executor disabled the same group is a k_flow launch whose continuation-operand prefetch
    buffers are sized by the host and covered by its shared memory."""
    import re

    from paper_2010_14962_b200 import Engine

    def leading_forests():
        with Engine(payload_path("cfg5_n120_p1_s5_m20_ext_bt"), device=-1, mode="ket") as e:
            text = e.describe()
        out = []
        for ln in text.splitlines():
            if not re.match(r"\s*\[\d+\] ", ln):
                continue
            m = re.search(r"forest .*units=(\d+) steps=(\d+) max_phases=(\d+)", ln)
            if not m or " deps=" in ln:
                break
            out.append(tuple(int(x) for x in m.groups()))
        return out

    # the group's 35 subtrees are spread over three concurrent launches by estimated time
    # (consumers of a light subtree no longer wait for the heaviest one)
    parts = leading_forests()
    assert len(parts) == 3, parts
    assert (sum(p[0] for p in parts), sum(p[1] for p in parts), max(p[2] for p in parts)) == (35, 617, 18)
    assert parts[0][2] < parts[2][2]  # light subtrees first, the deepest last
    monkeypatch.setenv("QCG_FOREST_SPLIT", "0")
    assert leading_forests() == [(35, 617, 18)]
    monkeypatch.delenv("QCG_FOREST_SPLIT")
    monkeypatch.setenv("QCG_NO_FOREST", "1")
    with Engine(payload_path("cfg5_n120_p1_s5_m20_ext_bt"), device=-1, mode="ket") as e:
        text = e.describe()
    tiles = [ln for ln in text.splitlines() if re.match(r"\s*\[\d+\] tiles ", ln)]
    assert tiles
    m = re.search(r"smem=(\d+) .*prefetch=(\d+)", tiles[0])
    assert m, tiles[0]
    smem, npre = int(m.group(1)), int(m.group(2))
    assert npre >= 1 and smem >= 256 * 16 + 2 * npre * 16


def test_final_reduction_fused_into_the_lead_gate(monkeypatch):
    """Config 5's last plan step is a gate whose result carries every batched slice bit (the
    lead rank-0 factor): the host planner marks it to do execute_plan's acc *= products and the
    slice sum in its epilogue (k_gate_reduce), so its 16 MB result is neither written nor
    re-read (the launch's algorithmic bytes drop by the tensor); QCG_FINAL_NO_FUSE=1 restores
    the separate walk."""
    import re

    from paper_2010_14962_b200 import Engine

    def last_gate():
        with Engine(payload_path("cfg5_n120_p1_s5_m20_ext_bt"), device=-1, mode="ket") as e:
            lines = [ln for ln in e.describe().splitlines() if re.match(r"\s*\[\d+\] gate ", ln)]
            return lines[-1], e.plan_stats()["moved_bytes"]

    fused, moved = last_gate()
    assert "+final" in fused and "plan_step=657" in fused, fused
    monkeypatch.setenv("QCG_FINAL_NO_FUSE", "1")
    plain, moved_plain = last_gate()
    assert "+final" not in plain
    b_f = float(re.search(r"bytes=([0-9.e+]+)", fused).group(1))
    b_p = float(re.search(r"bytes=([0-9.e+]+)", plain).group(1))
    assert abs((b_p - b_f) - 16 * 2 ** 20) <= 0.01 * 16 * 2 ** 20
    assert abs((moved_plain - moved) - 16 * 2 ** 20) <= 0.01 * 16 * 2 ** 20


def test_cfg1_cs_reference_run_serial_identity(oracle_mod):
    """The reference's own run_serial on the searched cut equals its GA-cut value, and the
    oracle reproduces the reference per slice on the searched cut."""
    rec = ref_json("cfg1_n20_p1_s1_m4_cs")
    want = cx(ref_json("cfg1_n20_p1_s1_m4")["run_serial"])
    assert abs(cx(rec["run_serial"]) - want) <= REL * abs(want)
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg1_n20_p1_s1_m4_cs")), "density")
    tot, per = net.sum_range(0, net.jobs, per_slice=True)
    ref = np.array([cx(v) for v in rec["slices"]])
    assert maxdiff(per, ref) <= REL
    assert abs(tot - want) <= REL * abs(want)


def test_cfg2_cs_oracle_vs_reference_range(oracle_mod):
    """N=60 at full size against the reference itself: 4096 density slices of the searched
    cut, per slice and summed."""
    rr = ref_json("cfg2_n60_p1_s1_m10_ext_cs")["ref_range"]
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg2_n60_p1_s1_m10_ext_cs")), "density")
    tot, per = net.sum_range(rr["lo"], rr["hi"], per_slice=True)
    ref = np.array([cx(v) for v in rr["slices"]])
    assert maxdiff(per, ref) <= REL
    assert abs(tot - cx(rr["sum_range"])) <= REL * np.abs(ref).sum()


def test_cfg2_cs_cross_cut_amplitude_on_oracle(oracle_mod):
    """|sum of all ket slices|^2 through the searched cut equals the GA cut's."""
    a = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg2_n60_p1_s1_m10_ext_cs")), "ket")
    r = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg2_n60_p1_s1_m10_ext_os")), "ket")
    sa = a.sum_range(0, a.jobs)
    sr = r.sum_range(0, r.jobs)
    assert abs(abs(sa) ** 2 - abs(sr) ** 2) <= REL * abs(sr) ** 2


def test_cfg4_cs_oracle_vs_reference_range(oracle_mod):
    rr = ref_json("cfg4_n100_p1_s1_m16_ext_cs")["ref_range"]
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg4_n100_p1_s1_m16_ext_cs")), "density")
    tot, per = net.sum_range(rr["lo"], rr["hi"], per_slice=True)
    ref = np.array([cx(v) for v in rr["slices"]])
    assert maxdiff(per, ref) <= REL
    assert abs(tot - cx(rr["sum_range"])) <= REL * np.abs(ref).sum()


# ----------------------------------------------------------------------------- GPU


@pytest.mark.gpu
def test_cfg2_cs_engine_vs_reference_and_oracle():
    """Density view: the reference's per-slice values at N=60; ket view: every slice vs the
    oracle, and |A|^2 equal to the GA cut's on the engine."""
    from paper_2010_14962_b200 import Engine
    from oracle import oracle as O

    stem = "cfg2_n60_p1_s1_m10_ext_cs"
    rr = ref_json(stem)["ref_range"]
    ref = np.array([cx(v) for v in rr["slices"]])
    with Engine(payload_path(stem), device=0, mode="density") as e:
        assert e.plan_stats()["peak_rank"] == 8
        assert maxdiff(e.slice_values(rr["lo"], rr["hi"]), ref) <= REL
        assert abs(e.sum_range(rr["lo"], rr["hi"]) - cx(rr["sum_range"])) <= REL * np.abs(ref).sum()
        p_density = e.run_serial()
    net = O.OracleNet(O.load_payload(payload_path(stem)), "ket")
    _, ka = net.sum_range(0, net.jobs, per_slice=True)
    with Engine(payload_path(stem), device=0, mode="ket") as e:
        vals = e.ket_values()
        p_cs = e.run_serial().real
    assert maxdiff(dephase(vals, ka), ka) <= REL
    with Engine(payload_path("cfg2_n60_p1_s1_m10_ext"), device=0, mode="ket") as e:
        p_ga = e.run_serial().real
    assert abs(p_cs - p_ga) <= REL * p_ga
    assert abs(p_density - p_ga) <= 1e-9 * p_ga  # all 4^10 density slices of the searched cut


@pytest.mark.gpu
def test_cfg3_cs_cross_cut_and_oracle():
    """Config 3 (QAOA p=2, N=50, k=14): two independently searched cuts (peaks 20 and 23)
    give the same |A|^2; ket slices vs the oracle; the reference's GA cut has no plan below
    peak 35, so cross-cut identity is the full-size pin."""
    from paper_2010_14962_b200 import Engine
    from oracle import oracle as O

    with Engine(payload_path("cfg3_n50_p2_s1_m14_cs"), device=0, mode="ket") as e:
        assert e.plan_stats()["peak_rank"] == 20
        a1 = e.ket_sum()
        v1 = e.ket_values(9000, 9064)
    with Engine(payload_path("cfg3_n50_p2_s1_m14_cs2"), device=0, mode="ket") as e:
        assert e.plan_stats()["peak_rank"] == 23
        a2 = e.ket_sum()
    assert abs(abs(a1) ** 2 - abs(a2) ** 2) <= REL * abs(a2) ** 2
    assert abs(a1 - a2) <= REL * abs(a2)  # same network tensors -> same global phase convention
    net = O.OracleNet(O.load_payload(payload_path("cfg3_n50_p2_s1_m14_cs")), "ket")
    _, ka = net.sum_range(9000, 9002, per_slice=True)
    assert maxdiff(dephase(v1[:2], ka), ka) <= REL


@pytest.mark.gpu
def test_cfg4_cs_engine_vs_reference_and_ga_cut():
    from paper_2010_14962_b200 import Engine

    stem = "cfg4_n100_p1_s1_m16_ext_cs"
    rr = ref_json(stem)["ref_range"]
    ref = np.array([cx(v) for v in rr["slices"]])
    with Engine(payload_path(stem), device=0, mode="density") as e:
        assert maxdiff(e.slice_values(rr["lo"], rr["hi"]), ref) <= REL
    for b in (0, 5):
        with Engine(payload_path(stem, b), device=0, mode="ket") as e:
            p_cs = e.run_serial().real
        with Engine(payload_path("cfg4_n100_p1_s1_m16_ext_os", b), device=0, mode="ket") as e:
            p_os = e.run_serial().real
        assert abs(p_cs - p_os) <= 1e-9 * p_os


@pytest.mark.gpu
def test_cfg5_cs_engine_vs_reference_and_ga_cut():
    """Config 5 (N=120, k=20): the reference's own density values on the searched cut, and
    the full amplitude against the GA cut through the order-searched plan (peak 20)."""
    from paper_2010_14962_b200 import Engine

    stem = "cfg5_n120_p1_s5_m20_ext_cs"
    rr = ref_json(stem)["ref_range"]
    ref = np.array([cx(v) for v in rr["slices"]])
    with Engine(payload_path(stem), device=0, mode="density") as e:
        assert maxdiff(e.slice_values(rr["lo"], rr["hi"]), ref) <= REL
    with Engine(payload_path(stem), device=0, mode="ket") as e:
        assert e.plan_stats()["peak_rank"] == 12
        a_cs = e.ket_sum()
    with Engine(payload_path("cfg5_n120_p1_s5_m20_ext_os"), device=0, mode="ket") as e:
        a_os = e.ket_sum()
    assert abs(abs(a_cs) ** 2 - abs(a_os) ** 2) <= 1e-9 * abs(a_os) ** 2


def density_from_ket(net, lo, hi):
    """Reference density ids [lo, hi) answered from the ket oracle: V(s) = A(k) conj(A(b)),
    digit i of s = 2 k_i + b_i (phase-free, so the oracle's own phase convention is fine)."""
    M = net.payload.M
    got = []
    for s in range(lo, hi):
        k = b = 0
        for i in range(M):
            d = (s >> (2 * (M - 1 - i))) & 3
            k, b = (k << 1) | (d >> 1), (b << 1) | (d & 1)
        got.append(net.sum_range(k, k + 1) * np.conj(net.sum_range(b, b + 1)))
    return np.array(got)


@pytest.mark.parametrize("stem", ["cfg5_n120_p1_s5_m20_ext_bt", "cfg2_n60_p1_s1_m10_ext_bt",
                                  "cfg4_n100_p1_s1_m16_ext_bt"])
def test_bt_oracle_vs_reference_range(oracle_mod, stem):
    """Batched-objective plans against the reference's own density values at full size (the
    ket-view oracle answers density ids exactly)."""
    rr = ref_json(stem)["ref_range"]
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path(stem)), "ket")
    ref = np.array([cx(v) for v in rr["slices"]])
    assert maxdiff(density_from_ket(net, rr["lo"], rr["hi"]), ref) <= REL


@pytest.mark.gpu
def test_cfg5_bt_engine_vs_reference_and_cs_cut():
    """Config 5 through the bench plan: the reference's density values (both views) and the
    full amplitude against the peak-objective cut (cross-cut identity)."""
    from paper_2010_14962_b200 import Engine

    stem = "cfg5_n120_p1_s5_m20_ext_bt"
    rr = ref_json(stem)["ref_range"]
    ref = np.array([cx(v) for v in rr["slices"]])
    with Engine(payload_path(stem), device=0, mode="density") as e:
        assert maxdiff(e.slice_values(rr["lo"], rr["hi"]), ref) <= REL
    with Engine(payload_path(stem), device=0, mode="ket") as e:
        assert e.plan_stats()["peak_rank"] == 12 and e.plan_stats()["batch_bits"] == 20
        assert maxdiff(e.slice_values(rr["lo"], rr["hi"]), ref) <= REL
        a_bt = e.ket_sum()
        a_bt2 = e.ket_sum()
        half = e.ket_sum(0, 1 << 19) + e.ket_sum(1 << 19, 1 << 20)
    assert a_bt == a_bt2  # bitwise reproducible
    assert abs(half - a_bt) <= REL * abs(a_bt)
    with Engine(payload_path("cfg5_n120_p1_s5_m20_ext_cs"), device=0, mode="ket") as e:
        a_cs = e.ket_sum()
    assert abs(a_bt - a_cs) <= REL * abs(a_cs)


@pytest.mark.gpu
@pytest.mark.parametrize("stem,other,nb", [("cfg2_n60_p1_s1_m10_ext_bt", "cfg2_n60_p1_s1_m10_ext", 1),
                                           ("cfg4_n100_p1_s1_m16_ext_bt", "cfg4_n100_p1_s1_m16_ext_os", 8)])
def test_bt_engine_vs_reference_and_other_cut(stem, other, nb):
    """Configs 2 and 4 through the batched-objective plans: the reference's density values
    (density view and ket view) and every bitstring's |A|^2 against the GA cut."""
    from paper_2010_14962_b200 import Engine

    rr = ref_json(stem)["ref_range"]
    ref = np.array([cx(v) for v in rr["slices"]])
    with Engine(payload_path(stem), device=0, mode="density") as e:
        assert maxdiff(e.slice_values(rr["lo"], rr["hi"]), ref) <= REL
    for b in range(nb):
        with Engine(payload_path(stem, b), device=0, mode="ket") as e:
            if b == 0:
                assert maxdiff(e.slice_values(rr["lo"], rr["hi"]), ref) <= REL
            p_bt = e.run_serial().real
        with Engine(payload_path(other, b), device=0, mode="ket") as e:
            p_o = e.run_serial().real
        assert abs(p_bt - p_o) <= 1e-9 * p_o, (b, p_bt, p_o)


@pytest.mark.gpu
def test_cfg3_bt_vs_cs_cut():
    from paper_2010_14962_b200 import Engine

    with Engine(payload_path("cfg3_n50_p2_s1_m14_bt"), device=0, mode="ket") as e:
        assert e.plan_stats()["peak_rank"] == ref_json("cfg3_n50_p2_s1_m14_bt")["cut_search"]["peak"] <= 24
        a_bt = e.ket_sum()
    with Engine(payload_path("cfg3_n50_p2_s1_m14_cs"), device=0, mode="ket") as e:
        a_cs = e.ket_sum()
    assert abs(a_bt - a_cs) <= REL * abs(a_cs)


def test_cut_search_tool_on_config1(tmp_path):
    """The search tool itself (oracle/_ref/cut_search, built here from the reference library):
    its FastPlan restatement is cross-checked against the reference's plan_from_order at
    start-up (exit code 3 on any mismatch), the emitted payload carries the reference's own
    plan for the reported cut, and both objectives keep M and bound the peak."""
    import os
    import subprocess

    from conftest import ROOT

    exe = os.path.join(ROOT, "oracle", "_ref", "cut_search")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/cut_search not built (needs the reference sources)")
    src = tmp_path / "cfg1.json"
    with gzip.open(payload_path("cfg1_n20_p1_s1_m4"), "rb") as f:
        src.write_bytes(f.read())
    for extra in ([], ["--objective", "batched", "--bound", "6"]):
        out = tmp_path / "out.json"
        r = subprocess.run([exe, "--payload", str(src), "--out", str(out), "--evals", "3000", "--threads", "2",
                            "--seed", "5", *extra], check=True, capture_output=True, text=True)
        rec = json.loads(r.stdout.strip().splitlines()[-1])
        p = json.loads(out.read_text())
        assert p["cut"] == rec["cut"] == sorted(p["cut"]) and len(p["cut"]) == rec["M"] == 4
        assert p["plan"]["peak_rank"] == rec["peak"] <= rec["reference_peak"]
        if extra:
            assert rec["peak"] <= 6 and rec["objective"] == "batched"
        # the emitted plan runs on the oracle and gives the reference's amplitude
        import oracle.oracle as O

        net = O.OracleNet(O.load_payload(str(out)), "density")
        want = cx(ref_json("cfg1_n20_p1_s1_m4")["run_serial"])
        assert abs(net.sum_range(0, net.jobs) - want) <= REL * abs(want)
