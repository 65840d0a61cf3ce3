"""A dense PlanStep inside the engine: the FP64 tensor-pipe GEMM (k_zgemm_dmma) as a pass launch.

The networks are the dense triangles of tools/dense_payload.py (payload rebuilt from a seed);
tests/golden/dense_triangle.ref.json holds the UNMODIFIED reference's run_serial and per-slice
values on exactly those payloads (tools/make_golden.py --dense). Anchors: execute_plan /
contract_pair (proj/core/src/contraction.cpp:288-319, 71-116) with M, K and N all large.
"""
import json

import numpy as np
import pytest

from conftest import cx, golden
from tools.dense_payload import dense_triangle, dense_value

CASES = [(5, 3, 3, 7), (4, 3, 3, 11), (6, 2, 3, 5)]
REL = 1e-10  # north_star tolerance


def build(case):
    a, b, c, seed = case
    pay, data = dense_triangle(a, b, c, seed)
    with open(golden("dense_triangle.ref.json")) as f:
        ref = json.load(f)[f"{a}_{b}_{c}_{seed}"]
    checksum = float(sum(np.sum(np.abs(d)) for d in data))
    assert abs(checksum - ref["checksum"]) <= 1e-9 * ref["checksum"], "payload generator drifted from the fixture"
    return json.dumps(pay, separators=(",", ":")).encode(), data, ref


@pytest.mark.parametrize("case", CASES, ids=[f"a{c[0]}b{c[1]}c{c[2]}" for c in CASES])
def test_reference_values_and_host_plan(oracle_mod, case, tmp_path):
    """The reference's run_serial equals the full numpy contraction, the pinned oracle is
    bit-identical to the reference per slice, and the host planner turns the dense step into
    a GEMM launch (the second step's 2^12-term sum too: it does not fit the dataflow tiles)."""
    from paper_2010_14962_b200 import Engine

    payload, data, ref = build(case)
    a, b, c, _ = case
    want = dense_value(a, b, c, data)
    assert abs(cx(ref["run_serial"]) - want) <= 1e-12 * abs(want)
    path = tmp_path / "dense.json"
    path.write_bytes(payload)
    net = oracle_mod.OracleNet(oracle_mod.load_payload(str(path)), "density")
    total, vals = net.sum_range(0, net.jobs, per_slice=True)
    assert np.array_equal(np.asarray(vals), np.array([cx(v) for v in ref["slices"]]))
    assert total == cx(ref["run_serial"])
    with Engine(payload, device=-1, mode="density", mem_budget_bytes=8 << 30) as e:
        text = e.describe()
        shapes = e.step_shapes()
    assert "(DMMA)" in text and f"M=2^{2 * c} N=2^{2 * b} K=2^{2 * (a - 1)} batch=2^2" in text, text
    assert [list(map(int, s)) for s in shapes] == ref["steps"]  # (rank_a, rank_b, shared, result_rank)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[f"a{c[0]}b{c[1]}c{c[2]}" for c in CASES])
def test_engine_matches_the_reference_through_the_gemm_launch(case):
    from paper_2010_14962_b200 import Engine

    payload, _, ref = build(case)
    want = np.array([cx(v) for v in ref["slices"]])
    with Engine(payload, device=0, mode="density") as e:
        kinds = [p["kind"] for p in e.profile_pass()]
        assert "k_zgemm_dmma" in kinds, kinds
        vals = e.slice_values(0, e.jobs())
        total = e.run_serial()
        again = e.slice_values(0, e.jobs())
    assert np.max(np.abs(vals - want)) <= REL * np.max(np.abs(want))
    assert abs(total - cx(ref["run_serial"])) <= REL * abs(cx(ref["run_serial"]))
    assert np.array_equal(vals, again)  # bitwise reproducible


@pytest.mark.gpu
def test_gemm_launch_against_the_dataflow_kernel(monkeypatch):
    """A/B inside the engine: the same dense step as k_flow tiles (QCG_NO_GEMM=1 keeps the
    first step there; the 2^12-term second step always takes the GEMM's k loop)."""
    from paper_2010_14962_b200 import Engine

    payload, _, ref = build(CASES[1])
    with Engine(payload, device=0, mode="density") as e:
        v_gemm = e.slice_values(0, e.jobs())
    monkeypatch.setenv("QCG_NO_GEMM", "1")
    try:
        with Engine(payload, device=0, mode="density") as e:
            v_flow = e.slice_values(0, e.jobs())
    except RuntimeError as ex:  # the dataflow kernel cannot hold this step at all
        assert "shared memory" in str(ex)
        return
    assert np.max(np.abs(v_gemm - v_flow)) <= 1e-12 * np.max(np.abs(v_gemm))


@pytest.mark.gpu
def test_gemm_launch_with_one_slice_per_pass():
    """The same dense network with no batched cut bits (max_batch_bits=0): the cut leg is fixed
    per pass by k_prep's gather and the GEMM launch runs with batch 1, four passes per call."""
    from paper_2010_14962_b200 import Engine

    payload, _, ref = build(CASES[0])
    want = np.array([cx(v) for v in ref["slices"]])
    with Engine(payload, device=0, mode="density", max_batch_bits=0) as e:
        st = e.plan_stats()
        assert st["batch_bits"] == 0 and st["chunks"] == 4
        assert "(DMMA)" in e.describe() and "batch=2^0" in e.describe()
        vals = e.slice_values(0, 4)
        total = e.run_serial()
        mid = e.sum_range(1, 3)
    assert np.max(np.abs(vals - want)) <= REL * np.max(np.abs(want))
    assert abs(total - cx(ref["run_serial"])) <= REL * abs(cx(ref["run_serial"]))
    assert abs(mid - (want[1] + want[2])) <= REL * np.max(np.abs(want))
