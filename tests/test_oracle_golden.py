"""The CPU oracle (oracle/qcut_oracle.c) pinned against the unmodified reference.

Golden values in tests/golden/ were produced by tools/make_golden.py from the
reference compiled from /root/reference (oracle/_ref/qcut_refgen).
"""
import numpy as np
import pytest

from conftest import RANDOM_STEMS, SMALL_QAOA, cx, payload_path, ref_json


def digits_to_ket_bra(s, M):
    k = b = 0
    for i in range(M):
        d = (s >> (2 * (M - 1 - i))) & 3
        k = (k << 1) | (d >> 1)
        b = (b << 1) | (d & 1)
    return k, b


@pytest.mark.parametrize("stem", SMALL_QAOA)
def test_density_oracle_matches_reference_per_slice(oracle_mod, stem):
    ref = ref_json(stem)
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path(stem)), "density")
    total, per = net.sum_range(0, net.jobs, per_slice=True)
    want = np.array([cx(v) for v in ref["slices"]])
    # same loop order as the reference: bit-identical per slice
    assert np.array_equal(per, want)
    assert total == cx(ref["run_serial"])


def test_readme_golden_value(oracle_mod):
    """proj/README.md:44-73: cut [17, 30], 16 jobs, peak 5, p = 0.0037456566518327397."""
    ref = ref_json("readme_n12_s7_m2")
    assert ref["info"]["cut"] == [17, 30]
    assert ref["info"]["plan"]["peak_rank"] == 5
    assert ref["run_serial"][0] == 0.0037456566518327397
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("readme_n12_s7_m2")), "density")
    assert net.jobs == 16
    assert net.sum_range(0, 16).real == 0.0037456566518327397


def test_config1_worked_example():
    """SURVEY §8(d) worked example (config 1, seed 1)."""
    info = ref_json("cfg1_n20_p1_s1_m4")["info"]
    assert info["gammas"] == [2.5909873700584827]
    assert info["betas"] == [0.020183603777160952]
    assert info["bitstrings"] == ["00100011101100000010"]
    assert info["cut"] == [10, 29, 64, 71]
    assert info["plan"]["peak_rank"] == 7
    assert ref_json("cfg1_n20_p1_s1_m4")["run_serial"][0] == 1.0593560561496424e-06


@pytest.mark.parametrize("stem", SMALL_QAOA + RANDOM_STEMS)
def test_ket_view_identity(oracle_mod, stem):
    """V(d) = A(k) conj(A(b)) per slice and p = |sum_k A(k)|^2 (SURVEY §8 parity identity)."""
    ref = ref_json(stem)
    p = oracle_mod.load_payload(payload_path(stem))
    net = oracle_mod.OracleNet(p, "ket")
    a, ka = net.sum_range(0, net.jobs, per_slice=True)
    want = cx(ref.get("run_serial", ref.get("serial")))
    assert abs(abs(a) ** 2 - want) <= 1e-12 * max(1e-300, abs(want)) + 1e-15
    M = p.M
    slices = np.array([cx(v) for v in ref["slices"]])
    got = np.array([ka[k] * np.conj(ka[b]) for k, b in (digits_to_ket_bra(s, M) for s in range(4 ** M))])
    assert np.max(np.abs(got - slices)) <= 1e-12 * max(1.0, np.max(np.abs(slices)))


@pytest.mark.parametrize("stem", RANDOM_STEMS)
def test_random_circuits_density(oracle_mod, stem):
    """test_contraction.cpp:178-188 style: plan value == reference run_serial (and dm_simulate)."""
    ref = ref_json(stem)
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path(stem)), "density")
    total, per = net.sum_range(0, net.jobs, per_slice=True)
    assert np.array_equal(per, np.array([cx(v) for v in ref["slices"]]))
    assert abs(total - cx(ref["serial"])) <= 1e-15
    assert abs(total - cx(ref["dm_simulate"])) <= 1e-10


@pytest.mark.parametrize("stem,want", [("cnot", 1.0), ("flip", 0.0)])
def test_cnot_cut_sums(oracle_mod, stem, want):
    """test_executor.cpp:67-80 (cut sum of a cnot circuit is 1) and the X+CNOT zero."""
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path(stem)), "density")
    assert net.jobs == 4
    assert abs(net.sum_range(0, 4) - want) < 1e-10
    assert abs(cx(ref_json(stem)["run_serial"]) - want) < 1e-10


def test_sum_range_split_additivity(oracle_mod):
    """test_executor.cpp:92-99."""
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path("cfg1_n20_p1_s1_m4")), "density")
    whole = net.sum_range(0, 256)
    split = net.sum_range(0, 100) + net.sum_range(100, 256)
    assert abs(whole - split) < 1e-18
    with pytest.raises(ValueError):
        net.sum_range(2, 1)
    with pytest.raises(ValueError):
        net.sum_range(0, 257)


def test_contract_pair_known_answers(oracle_mod):
    """test_contraction.cpp:46-106: delta identity, H on |0><0|, matrix product, leg order."""
    O = oracle_mod
    rho0 = np.array([1, 0, 0, 0], dtype=complex)
    delta = np.zeros(16, dtype=complex)
    for s in range(4):
        delta[s * 4 + s] = 1
    assert np.array_equal(O.contract_pair(4, rho0, [0], delta, [0]), rho0)
    s2 = 1 / np.sqrt(2)
    H = np.array([[s2, s2], [s2, -s2]])
    gt = np.zeros(16, dtype=complex)
    for s in range(4):
        for t in range(4):
            gt[s * 4 + t] = H[t // 2][s // 2] * np.conj(H[t % 2][s % 2])
    assert np.allclose(O.contract_pair(4, rho0, [0], gt, [0]), 0.5, atol=1e-12)
    rng = np.random.default_rng(2)
    a = rng.uniform(-1, 1, 16) + 1j * rng.uniform(-1, 1, 16)
    b = rng.uniform(-1, 1, 16) + 1j * rng.uniform(-1, 1, 16)
    A, B = a.reshape(4, 4), b.reshape(4, 4)
    assert np.allclose(O.contract_pair(4, a, [1], b, [0]).reshape(4, 4), A @ B, atol=1e-12)
    assert np.allclose(O.contract_pair(4, a, [0], b, [0]).reshape(4, 4), A.T @ B, atol=1e-12)
    with pytest.raises(ValueError):
        O.contract_pair(4, a, [5], b, [0])
    with pytest.raises(ValueError):
        O.contract_pair(4, a, [0, 0], b, [0, 1])
