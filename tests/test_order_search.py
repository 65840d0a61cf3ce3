"""plans from a searched elimination order (oracle/_ref/order_search, fed
through the reference's own plan_from_order, contraction.cpp:118-262).

An *_os payload keeps its source's network and cut and replaces only the plan. The
contraction order changes nothing but rounding, so every ket slice value must agree with
the source plan's to 1e-10 (CPU: the oracle on both plans; GPU: the engine on the *_os
plan against the oracle and against the engine on the reference plan).
"""
import gzip
import json

import numpy as np
import pytest

from conftest import payload_path, ref_json

REL = 1e-10
OS = {  # os stem -> (source stem, bitstrings)
    "cfg2_n60_p1_s1_m10_ext_os": ("cfg2_n60_p1_s1_m10_ext", 1),
    "cfg4_n100_p1_s1_m16_ext_os": ("cfg4_n100_p1_s1_m16_ext", 8),
    "cfg5_n120_p1_s5_m20_ext_os": ("cfg5_n120_p1_s5_m20_ext", 1),
}


def load(stem, b=0):
    with gzip.open(payload_path(stem, b), "rt") as f:
        return json.load(f)


def maxdiff(a, ref):
    return np.max(np.abs(a - ref)) / np.abs(ref).max()


@pytest.mark.parametrize("stem", sorted(OS))
def test_os_payload_keeps_network_and_cut(stem):
    src, nb = OS[stem]
    rec = ref_json(stem)["order_search"]
    for b in range(nb):
        p, q = load(stem, b), load(src, b)
        assert p["network"] == q["network"] and p["cut"] == q["cut"] and p["v"] == q["v"]
        assert len(p["plan"]["steps"]) == len(q["plan"]["steps"]) == rec["steps"]
    assert p["plan"]["peak_rank"] == rec["peak"] < q["plan"]["peak_rank"] == rec["reference_peak"]
    assert p["plan"]["cost_estimate"] < q["plan"]["cost_estimate"]


@pytest.mark.parametrize("stem", sorted(OS))
def test_os_plan_host_program_valid(stem):
    from paper_2010_14962_b200 import Engine

    with Engine(payload_path(stem), device=-1, mode="ket") as e:
        st = e.plan_stats()
    with Engine(payload_path(OS[stem][0]), device=-1, mode="ket") as e:
        st_ref = e.plan_stats()
    assert st["peak_rank"] == ref_json(stem)["order_search"]["peak"]
    assert st["flops"] < st_ref["flops"] and st["essential_bytes"] < st_ref["essential_bytes"]


def test_cfg2_os_plan_equivalent_on_oracle(oracle_mod):
    """Every ket slice of config 2 through both plans on the CPU oracle."""
    a = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg2_n60_p1_s1_m10_ext_os")), "ket")
    r = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg2_n60_p1_s1_m10_ext")), "ket")
    sa, va = a.sum_range(0, a.jobs, per_slice=True)
    sr, vr = r.sum_range(0, r.jobs, per_slice=True)
    assert maxdiff(va, vr) <= REL
    assert abs(sa - sr) <= REL * abs(sr)


def test_cfg4_os_plan_equivalent_on_oracle(oracle_mod):
    a = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg4_n100_p1_s1_m16_ext_os", 3)), "ket")
    r = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg4_n100_p1_s1_m16_ext", 3)), "ket")
    _, va = a.sum_range(77, 78, per_slice=True)
    _, vr = r.sum_range(77, 78, per_slice=True)
    assert maxdiff(va, vr) <= REL


@pytest.mark.gpu
def test_cfg2_os_engine_vs_oracle():
    from paper_2010_14962_b200 import Engine
    from oracle import oracle as O

    net = O.OracleNet(O.load_payload(payload_path("cfg2_n60_p1_s1_m10_ext")), "ket")
    a_ref, ka = net.sum_range(0, net.jobs, per_slice=True)
    with Engine(payload_path("cfg2_n60_p1_s1_m10_ext_os"), device=0, mode="ket") as e:
        assert e.plan_stats()["peak_rank"] == 11
        vals = e.ket_values()
        c = np.vdot(vals, ka)
        assert maxdiff(vals * (c / abs(c)), ka) <= REL
        assert abs(e.run_serial().real - abs(a_ref) ** 2) <= REL * abs(a_ref) ** 2


@pytest.mark.gpu
def test_cfg4_os_engine_vs_reference_plan():
    """All 8 bitstrings' full amplitudes through both plans on the engine."""
    from paper_2010_14962_b200 import Engine

    for b in (0, 5):
        with Engine(payload_path("cfg4_n100_p1_s1_m16_ext_os", b), device=0, mode="ket") as e:
            p_os = e.run_serial().real
            v_os = e.ket_values(1000, 1064)
        with Engine(payload_path("cfg4_n100_p1_s1_m16_ext", b), device=0, mode="ket") as e:
            p_ref = e.run_serial().real
            v_ref = e.ket_values(1000, 1064)
        assert abs(p_os - p_ref) <= 1e-9 * p_ref
        c = np.vdot(v_os, v_ref)
        assert maxdiff(v_os * (c / abs(c)), v_ref) <= REL


@pytest.mark.gpu
def test_cfg5_os_engine_vs_reference_plan_and_oracle():
    """Config 5 (N=120, k=20): the peak-20 plan against the reference's peak-30 plan on the
    engine (64 ket slices), and against the oracle on 2 slices."""
    from paper_2010_14962_b200 import Engine
    from oracle import oracle as O

    with Engine(payload_path("cfg5_n120_p1_s5_m20_ext_os"), device=0, mode="ket") as e:
        assert e.plan_stats()["peak_rank"] == 20
        v_os = e.ket_values(4096, 4160)
    net = O.OracleNet(O.load_payload(payload_path("cfg5_n120_p1_s5_m20_ext_os")), "ket")
    _, ka = net.sum_range(4096, 4098, per_slice=True)
    c = np.vdot(v_os[:2], ka)
    assert np.max(np.abs(v_os[:2] * (c / abs(c)) - ka)) <= REL * np.abs(ka).max()
    with Engine(payload_path("cfg5_n120_p1_s5_m20_ext"), device=0, mode="ket") as e:
        v_ref = e.ket_values(4096, 4160)
    c = np.vdot(v_os, v_ref)
    assert maxdiff(v_os * (c / abs(c)), v_ref) <= REL


# ---- opt-in 2-qubit operator-Schmidt split (order_search --split-2q 1) ----
# The split keeps every original edge id, so the cut and the slice enumeration are the
# source's: every slice value must match the unsplit network's.


def test_split_payload_keeps_cut_and_reference_value():
    from conftest import cx

    p, q = load("cfg1_n20_p1_s1_m4_split"), load("cfg1_n20_p1_s1_m4")
    assert p["cut"] == q["cut"]
    rec = ref_json("cfg1_n20_p1_s1_m4_split")
    assert rec["order_search"]["split_2q"] == 30  # the 30 ZZ gates of the N=20 3-regular graph
    want = cx(ref_json("cfg1_n20_p1_s1_m4")["run_serial"])
    assert abs(cx(rec["run_serial"]) - want) <= REL * abs(want)  # the reference's own run_serial


def test_split_density_slices_on_oracle(oracle_mod):
    """Every density slice of config 1 through the split network (oracle) vs the reference's
    per-slice values of the original network."""
    from conftest import cx

    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg1_n20_p1_s1_m4_split")), "density")
    _, per = net.sum_range(0, net.jobs, per_slice=True)
    want = np.array([cx(v) for v in ref_json("cfg1_n20_p1_s1_m4")["slices"]])
    assert maxdiff(per, want) <= REL


def test_cfg2_split_ket_slices_on_oracle(oracle_mod):
    a = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg2_n60_p1_s1_m10_ext_split")), "ket")
    r = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg2_n60_p1_s1_m10_ext")), "ket")
    _, va = a.sum_range(0, a.jobs, per_slice=True)
    _, vr = r.sum_range(0, r.jobs, per_slice=True)
    c = np.vdot(va, vr)
    assert maxdiff(va * (c / abs(c)), vr) <= REL


@pytest.mark.gpu
def test_split_networks_on_engine():
    from conftest import cx
    from paper_2010_14962_b200 import Engine
    from oracle import oracle as O

    want = cx(ref_json("cfg1_n20_p1_s1_m4")["run_serial"])
    for mode in ("density", "ket"):
        with Engine(payload_path("cfg1_n20_p1_s1_m4_split"), device=0, mode=mode) as e:
            got = e.run_serial()
            assert abs(got - want) <= REL * abs(want)
            if mode == "density":
                per = e.slice_values(0, 256)
                ref = np.array([cx(v) for v in ref_json("cfg1_n20_p1_s1_m4")["slices"]])
                assert maxdiff(per, ref) <= REL
    net = O.OracleNet(O.load_payload(payload_path("cfg2_n60_p1_s1_m10_ext")), "ket")
    _, ka = net.sum_range(0, net.jobs, per_slice=True)
    with Engine(payload_path("cfg2_n60_p1_s1_m10_ext_split"), device=0, mode="ket") as e:
        assert e.plan_stats()["peak_rank"] == 10
        vals = e.ket_values()
    c = np.vdot(vals, ka)
    assert maxdiff(vals * (c / abs(c)), ka) <= REL


@pytest.mark.gpu
def test_density_view_at_scale():
    """The reference's own density view at scale: config 2 through the
    peak-11 plan (22-bit density tensors, 4^10 density slices; the whole amplitude takes
    ~200 s on one B200 vs ~1.4e5 s for the reference on 8 cores). An unaligned 5000-slice
    range against the ket view's exact answer for density ids, V(s) = A(k) conj(A(b))."""
    from paper_2010_14962_b200 import Engine

    with Engine(payload_path("cfg2_n60_p1_s1_m10_ext_os"), device=0, mode="ket") as e:
        kv = np.abs(e.ket_values())
        nz = np.flatnonzero(kv > 0.1 * kv.max())  # ket slices with A(k) != 0 (ZZ structure zeroes many)
        ka, kb, M = int(nz[0]), int(nz[-1]), e.M
        s = sum((2 * ((ka >> (M - 1 - i)) & 1) + ((kb >> (M - 1 - i)) & 1)) << (2 * (M - 1 - i)) for i in range(M))
        lo = max(0, s - 1000)
        hi = lo + 5000
        k = e.sum_range(lo, hi)
        kper = e.slice_values(s, s + 64)
    with Engine(payload_path("cfg2_n60_p1_s1_m10_ext_os"), device=0, mode="density") as e:
        d = e.sum_range(lo, hi)
        per = e.slice_values(s, s + 64)
    assert abs(kper[0]) > 0
    assert abs(d - k) <= REL * np.abs(kper).max() * 5000
    assert maxdiff(per, kper) <= REL
