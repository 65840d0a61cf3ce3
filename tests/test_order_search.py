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
