"""contract_pair on the device (qc_contract_pair) against the reference's own results.

Anchors: qcut::contract_pair (proj/core/src/contraction.cpp:71-116) and its tests
(proj/tests/test_contraction.cpp:46-134). tests/golden/pairs.npz holds seeded operands and
the result of the UNMODIFIED reference per case (tools/make_golden.py --pairs, refgen pair).
The oracle's restatement must reproduce them bit for bit (CPU test); the device paths --
the FP64 tensor-pipe GEMM (DMMA), its DFMA partner and the thin-shape kernel -- must match to
1e-12 of the result's largest entry (the GEMM sums in a different order than the
reference's sequential s loop, so bit equality is not expected; 1e-12 << north_star's 1e-10).
"""
import numpy as np
import pytest

from conftest import golden
from paper_2010_14962_b200 import RankGuardError, contract_pair, contract_pair_bench

TOL = 1e-12


def cases():
    z = np.load(golden("pairs.npz"))
    out = []
    i = 0
    while f"spec{i}" in z:
        spec = z[f"spec{i}"].tolist()
        ra, rb, k = spec[:3]
        out.append((i, ra, spec[3:3 + k], rb, spec[3 + k:3 + 2 * k], z[f"a{i}"], z[f"b{i}"], z[f"out{i}"]))
        i += 1
    return out


CASES = cases()


def test_fixture_covers_the_reference_shapes():
    assert len(CASES) == 10
    shapes = {(c[1], len(c[2])) for c in CASES}
    assert (4, 2) in shapes and (6, 3) in shapes  # BM_ContractPair, bench_main.cpp:60-62


@pytest.mark.parametrize("case", CASES, ids=[f"pair{c[0]}" for c in CASES])
def test_oracle_is_bit_identical_to_the_reference(oracle_mod, case):
    _, ra, la, rb, lb, a, b, want = case
    got = oracle_mod.contract_pair(4, a, la, b, lb)
    assert np.array_equal(got, want)


def test_argument_checks_match_the_reference_without_a_device():
    """contraction.cpp:74-87 / test_contraction.cpp:108-134: the checks run on the host, before
    any device call, with the reference's messages."""
    rng = np.random.default_rng(4)
    a = rng.uniform(-1, 1, 16) + 0j
    b = rng.uniform(-1, 1, 16) + 0j
    with pytest.raises(ValueError, match="needs at least one shared leg"):
        contract_pair(a, [], b, [])
    with pytest.raises(ValueError, match="shared leg lists differ in length: 2 vs 1"):
        contract_pair(a, [0, 1], b, [0])
    with pytest.raises(ValueError, match=r"leg 5 out of range for rank-2 tensor \(left\)"):
        contract_pair(a, [5], b, [0])
    with pytest.raises(ValueError, match=r"leg 0 repeated \(left\)"):
        contract_pair(a, [0, 0], b, [0, 1])
    with pytest.raises(ValueError, match=r"leg 7 out of range for rank-2 tensor \(right\)"):
        contract_pair(a, [0], b, [7])
    a3 = rng.uniform(-1, 1, 64) + 0j
    with pytest.raises(RankGuardError) as ei:
        contract_pair(a3, [2], a3, [0], max_rank=3)  # result rank 4 > 3
    assert ei.value.rank == 4 and ei.value.max_rank == 3
    assert "rank-4" in str(ei.value) and "max rank 3" in str(ei.value)
    with pytest.raises(ValueError, match="GEMM paths need"):
        contract_pair(a, [1], b, [0], path="dmma")  # K = 4: not a dense contraction


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    a = np.ones(16, dtype=complex)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        contract_pair(a, [1], a, [0])


def _paths(ra, rb, k, dim=4):
    K = dim ** k
    ps = ["auto", "small"]
    if K >= 8:
        ps += ["dmma", "dfma"]
    return ps


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[f"pair{c[0]}" for c in CASES])
def test_device_paths_match_the_reference(case):
    _, ra, la, rb, lb, a, b, want = case
    scale = np.max(np.abs(want))
    for path in _paths(ra, rb, len(la)):
        got = contract_pair(a, la, b, lb, max_rank=30, path=path)
        assert got.shape == want.shape
        assert np.max(np.abs(got - want)) <= TOL * scale, (path, np.max(np.abs(got - want)) / scale)


@pytest.mark.gpu
def test_known_answers():
    """test_contraction.cpp:46-106 on the device: delta identity, H on |0><0|, matrix product,
    leg order on both operands."""
    rho0 = np.array([1, 0, 0, 0], dtype=complex)
    delta = np.zeros(16, dtype=complex)
    for s in range(4):
        delta[s * 4 + s] = 1
    assert np.array_equal(contract_pair(rho0, [0], delta, [0]), rho0)
    s2 = 1 / np.sqrt(2)
    H = np.array([[s2, s2], [s2, -s2]])
    gt = np.zeros(16, dtype=complex)
    for s in range(4):
        for t in range(4):
            gt[s * 4 + t] = H[t // 2][s // 2] * np.conj(H[t % 2][s % 2])
    assert np.allclose(contract_pair(rho0, [0], gt, [0]), 0.5, atol=1e-12)
    rng = np.random.default_rng(2)
    a = rng.uniform(-1, 1, 16) + 1j * rng.uniform(-1, 1, 16)
    b = rng.uniform(-1, 1, 16) + 1j * rng.uniform(-1, 1, 16)
    A, B = a.reshape(4, 4), b.reshape(4, 4)
    assert np.allclose(contract_pair(a, [1], b, [0]).reshape(4, 4), A @ B, atol=1e-12)
    assert np.allclose(contract_pair(a, [0], b, [0]).reshape(4, 4), A.T @ B, atol=1e-12)
    a5 = rng.uniform(-1, 1, 4 ** 5) + 0j
    g = contract_pair(a5, [3, 4], a5, [0, 1])  # rank arithmetic, test_contraction.cpp:64-71
    assert g.size == 4 ** 6


@pytest.mark.gpu
@pytest.mark.parametrize("spec", [(8, [4, 5, 6, 7], 8, [0, 1, 2, 3], 4), (7, [6, 0, 3], 6, [1, 5, 2], 4),
                                  (12, [9, 10, 11], 11, [0, 1, 2], 2), (13, [0, 5, 9, 12, 3], 9, [8, 1, 0, 4, 6], 2),
                                  (3, [2], 14, [7], 2), (16, [15, 14, 13, 12], 4, [0, 1, 2, 3], 2)],
                         ids=["bm_8_4", "dim4_mixed", "dim2_gemm", "dim2_mixed", "dim2_thin", "dim2_n1"])
def test_larger_shapes_against_the_oracle(oracle_mod, spec):
    """BM_ContractPair's (8, 4) shape, mixed leg orders and the binary view (dim 2), every
    applicable path, against the pinned oracle."""
    ra, la, rb, lb, dim = spec
    rng = np.random.default_rng(ra * 100 + rb)
    a = rng.uniform(-1, 1, dim ** ra) + 1j * rng.uniform(-1, 1, dim ** ra)
    b = rng.uniform(-1, 1, dim ** rb) + 1j * rng.uniform(-1, 1, dim ** rb)
    want = oracle_mod.contract_pair(dim, a, la, b, lb)
    scale = np.max(np.abs(want))
    for path in _paths(ra, rb, len(la), dim):
        got = contract_pair(a, la, b, lb, max_rank=40, dim=dim, path=path)
        assert np.max(np.abs(got - want)) <= TOL * scale, (path, np.max(np.abs(got - want)) / scale)


@pytest.mark.gpu
def test_full_size_shape_by_linearity_and_bench_hook():
    """BM_ContractPair's largest shape (9, 4) (M = N = 1024, K = 256): too slow to loop over on
    the oracle in a test, so it is checked through size-independent properties -- linearity in
    each operand and agreement of the tensor-pipe and FMA-pipe kernels -- plus 64 result rows
    recomputed with numpy from the permuted operands. The bench hook returns the same tensor."""
    rng = np.random.default_rng(94)
    n = 4 ** 9
    a1 = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    a2 = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    b = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    la, lb = [5, 6, 7, 8], [0, 1, 2, 3]
    c1 = contract_pair(a1, la, b, lb, max_rank=30, path="dmma")
    c2 = contract_pair(a2, la, b, lb, max_rank=30, path="dmma")
    c12 = contract_pair(a1 + (0.5 - 2j) * a2, la, b, lb, max_rank=30, path="dmma")
    scale = np.max(np.abs(c12))
    assert np.max(np.abs(c12 - (c1 + (0.5 - 2j) * c2))) <= 1e-11 * scale
    cf = contract_pair(a1, la, b, lb, max_rank=30, path="dfma")
    assert np.max(np.abs(cf - c1)) <= TOL * np.max(np.abs(c1))
    A, B = a1.reshape(1024, 256), b.reshape(256, 1024)
    rows = rng.choice(1024, 64, replace=False)
    assert np.max(np.abs(c1.reshape(1024, 1024)[rows] - A[rows] @ B)) <= 1e-11 * np.max(np.abs(c1))
    r = contract_pair_bench(a1, la, b, lb, path="auto", reps=3, warmup=1)
    assert r["path"] == "dmma" and r["kernel_ms"] > 0 and r["e2e_ms"] >= r["kernel_ms"]
    assert np.array_equal(r["out"], c1)  # same kernel, same order: bitwise reproducible
