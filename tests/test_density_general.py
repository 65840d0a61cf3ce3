"""General density mode: mixed inputs and non-projector POVM elements.

Fixtures `mixed_*` (tools/make_golden.py --mixed, `qcut_refgen mixed`): the reference test
generator's random circuits (proj/tests/helpers.hpp random_circuit) with rho = w|a><a| +
(1-w)|b><b| inputs and E = u|0><0| + v|psi><psi| measurements (circuit.hpp:62-79), a random
cut, the reference's run_serial, dm_simulate and every per-slice value sum_range(s, s+1)
(executor.cpp:45-68). Such tensors do not factorise as K (x) conj(K): only the density view
runs them.
"""
import glob
import os

import numpy as np
import pytest

from conftest import GOLD, cx, payload_path, ref_json

MIXED = sorted(os.path.basename(p)[: -len(".ref.json")] for p in glob.glob(os.path.join(GOLD, "mixed_*.ref.json")))
REL = 1e-10


def test_fixtures_exist():
    assert len(MIXED) >= 3


@pytest.mark.parametrize("stem", MIXED)
def test_reference_matches_dm_simulate(stem):
    """The reference's sliced contraction equals its dense density-matrix simulator."""
    ref = ref_json(stem)
    assert abs(cx(ref["serial"]) - cx(ref["dm_simulate"])) <= 1e-12 * abs(cx(ref["dm_simulate"]))
    assert abs(sum(cx(v) for v in ref["slices"]) - cx(ref["serial"])) <= 1e-12 * abs(cx(ref["serial"]))


@pytest.mark.parametrize("stem", MIXED)
def test_oracle_density_view_per_slice(oracle_mod, stem):
    """The oracle's density view (the same loop order as contract_pair) is bit-identical per slice."""
    ref = ref_json(stem)
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path(stem)), "density")
    total, per = net.sum_range(0, net.jobs, per_slice=True)
    assert np.array_equal(per, np.array([cx(v) for v in ref["slices"]]))
    assert total == cx(ref["serial"])


@pytest.mark.parametrize("stem", MIXED)
def test_ket_view_refuses_non_factorising(stem):
    """The ket view needs pure inputs and projector measurements: QC_EINVAL -> ValueError."""
    from paper_2010_14962_b200 import Engine

    with pytest.raises(ValueError, match="factorise"):
        Engine(payload_path(stem), device=-1, mode="ket")


@pytest.mark.gpu
@pytest.mark.parametrize("stem", MIXED)
def test_engine_density_view_matches_reference(stem):
    """Every slice and the total of the engine's dim-4 view against the reference (1e-10),
    through full, partial and per-pass-split ranges."""
    from paper_2010_14962_b200 import Engine

    ref = ref_json(stem)
    want = np.array([cx(v) for v in ref["slices"]])
    scale = max(1e-300, np.max(np.abs(want)))
    for cap in (-1, 2):  # all slices in one pass; then 4 slices per pass (many passes)
        with Engine(payload_path(stem), device=0, mode="density", max_batch_bits=cap) as e:
            got = e.slice_values(0, e.jobs())
            assert np.max(np.abs(got - want)) <= REL * scale, (stem, cap)
            p = e.run_serial()
            assert abs(p - cx(ref["serial"])) <= REL * abs(cx(ref["serial"])), (stem, cap, p)
            lo, hi = 3, e.jobs() - 5
            assert abs(e.sum_range(lo, hi) - want[lo:hi].sum()) <= REL * np.sum(np.abs(want))
