"""Amplitude-level parity for the headline workload and configs 2-5.

Fixtures (tools/make_golden.py --amplitudes, from the compiled reference and the pinned
oracle; nothing here reads /root/reference):

* ``amplitudes.json``: per (plan, bitstring) the oracle's ket amplitude A = sum_k A(k)
  over EVERY slice (qcut_oracle.c, the restatement of sum_range -> execute_plan ->
  contract_pair, executor.cpp:45-70), |A|^2, sum |A(k)|^2, a weighted checksum of all
  2^M slice values and 64 largest + 64 strided slice values with their ids. Every
  network is pinned through two independent cuts where affordable (a cut only splits the
  same contraction, cutting.hpp:41-46): the oracle values agree across cuts.
* ``cfg5_n120_p1_s5_m20_ext_bt.refslices.json``: the compiled reference's own
  density-slice values sum_range(s, s+1) on 320 ids of the headline plan.

GPU tests compare the engine (through the C-ABI) with these at 1e-10 relative
(BASELINE north star); CPU tests pin the fixtures themselves.
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLD, cx, payload_path

REL = 1e-10
AMPS = json.load(open(os.path.join(GOLD, "amplitudes.json")))
REFSL = json.load(open(os.path.join(GOLD, "cfg5_n120_p1_s5_m20_ext_bt.refslices.json")))
KEYS = sorted(AMPS)
HEADLINE = "cfg5_n120_p1_s5_m20_ext_bt"


def split_key(key):
    stem, b = key.rsplit(".b", 1)
    return stem, int(b)


def density_id(k, b, M):
    """Density slice id of the ket pair (k, b): digit i = 2 k_i + b_i, MSB = first cut edge
    (cutting.cpp:41-52, SURVEY §8 conventions)."""
    return sum(((((k >> (M - 1 - i)) & 1) << 1) | ((b >> (M - 1 - i)) & 1)) << (2 * (M - 1 - i)) for i in range(M))


# ---------------------------------------------------------------- CPU: the fixtures themselves


def test_fixture_cross_cut_agreement():
    """The oracle's amplitude of one (network, bitstring) agrees across independent cuts."""
    by_net = {}
    for key, r in AMPS.items():
        by_net.setdefault((r["network"], r["bitstring"]), []).append(cx(r["A"]))
    multi = 0
    for (net, b), vals in by_net.items():
        assert abs(vals[0]) > 0, (net, b)
        for v in vals[1:]:
            multi += 1
            assert abs(v - vals[0]) <= REL * abs(vals[0]), (net, b, v, vals[0])
    assert multi >= 10  # cfg5 (bt/cs), cfg4 x 8 (bt/cs), cfg2 (bt/reference plan)


@pytest.mark.parametrize("key", [k for k in KEYS if AMPS[k]["M"] <= 20])
def test_fixture_slices_match_oracle(oracle_mod, key):
    """Re-run the oracle on the fixture's strided and top slices (a few ms each)."""
    stem, b = split_key(key)
    r = AMPS[key]
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path(stem, b)), "ket")
    ids = r["strided_ids"][:8] + r["top_ids"][:8]
    want = [cx(v) for v in r["strided_vals"][:8] + r["top_vals"][:8]]
    for i, w in zip(ids, want):
        got = net.sum_range(i, i + 1)
        assert abs(got - w) <= 1e-12 * max(abs(w), 1e-300), (key, i, got, w)


def test_refslices_are_ket_products():
    """The reference's density slices V(d(k, b)) equal A(k) conj(A(b)) of the oracle's ket
    slices (SURVEY §8 parity identity) on the 256 (k, b) pairs of the 16 largest ket slices."""
    r = AMPS[HEADLINE + ".b0"]
    M = r["M"]
    top = r["top_ids"][:16]
    tv = [cx(v) for v in r["top_vals"][:16]]
    ids = REFSL["ids"]
    vals = [cx(v) for v in REFSL["slices"]]
    scale = max(abs(v) for v in vals)
    for i in range(16):
        for j in range(16):
            n = 16 * i + j
            assert ids[n] == density_id(top[i], top[j], M)
            want = tv[i] * tv[j].conjugate()
            assert abs(vals[n] - want) <= REL * scale, (i, j, vals[n], want)


def test_refslices_density_oracle(oracle_mod):
    """Two of the reference's density slices re-computed by the oracle's density view."""
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path(HEADLINE)), "density")
    for n in (0, 17):
        s = REFSL["ids"][n]
        got = net.sum_range(s, s + 1)
        want = cx(REFSL["slices"][n])
        assert abs(got - want) <= 1e-12 * abs(want), (s, got, want)


# ---------------------------------------------------------------- GPU: the engine


@pytest.fixture(scope="module")
def Engine():
    from paper_2010_14962_b200 import Engine as E

    return E


def check_values(key, vals):
    r = AMPS[key]
    scale = max(abs(cx(v)) for v in r["top_vals"])
    k = np.arange(len(vals), dtype=np.float64)
    w = np.cos(0.7 * k)
    A = complex(math.fsum(vals.real), math.fsum(vals.imag))
    want = cx(r["A"])
    assert abs(A - want) <= REL * abs(want), (key, A, want)
    assert abs(math.fsum(np.abs(vals) ** 2) - r["sum_abs2"]) <= REL * r["sum_abs2"]
    chk = complex(math.fsum(w * vals.real), math.fsum(w * vals.imag))
    want_chk = cx(r["checksum_cos07"])
    assert abs(chk - want_chk) <= REL * math.sqrt(r["sum_abs2"] * len(vals)), (key, chk, want_chk)
    for ids, vs in ((r["top_ids"], r["top_vals"]), (r["strided_ids"], r["strided_vals"])):
        got = vals[np.array(ids)]
        assert np.max(np.abs(got - np.array([cx(v) for v in vs]))) <= REL * scale, key


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_engine_amplitude(Engine, key):
    """The engine's amplitude (device-reduced) and every slice value against the oracle's."""
    stem, b = split_key(key)
    want = cx(AMPS[key]["A"])
    with Engine(payload_path(stem, b), device=0, mode="ket") as e:
        a = e.ket_sum()
        assert abs(a - want) <= REL * abs(want), (key, a, want)
        p = e.run_serial()  # |sum_k A(k)|^2 = the reference's run_serial (density view)
        assert abs(p.real - abs(want) ** 2) <= REL * abs(want) ** 2 and p.imag == 0.0
        check_values(key, e.ket_values())


@pytest.mark.gpu
@pytest.mark.parametrize("stem", ["cfg5_n120_p1_s5_m20_ext_os", "cfg4_n100_p1_s1_m16_ext_os"])
def test_engine_amplitude_other_plans(Engine, stem):
    """Order-searched plans on the GA cut (peak 20 / 18): same amplitude as the oracle's
    through the searched cuts (cut-independent, cutting.hpp:41-46)."""
    src = stem.replace("_os", "_bt")
    want = cx(AMPS[src + ".b0"]["A"])
    with Engine(payload_path(stem, 0), device=0, mode="ket") as e:
        a = e.ket_sum()
    assert abs(a - want) <= REL * abs(want), (stem, a, want)


@pytest.mark.gpu
def test_engine_refslices_ket_view(Engine):
    """All 320 reference density slices of the headline plan from the engine's ket view."""
    ids = REFSL["ids"]
    want = np.array([cx(v) for v in REFSL["slices"]])
    scale = np.max(np.abs(want))
    with Engine(payload_path(HEADLINE), device=0, mode="ket") as e:
        got = np.array([e.slice_values(s, s + 1)[0] for s in ids])
        # partial-range sum_range semantics on a block of 4 ids around the first one
        s0 = ids[0] & ~3
        blk = e.sum_range(s0, s0 + 4)
        assert abs(blk - e.slice_values(s0, s0 + 4).sum()) <= REL * scale
    assert np.max(np.abs(got - want)) <= REL * scale


@pytest.mark.gpu
def test_engine_refslices_density_view(Engine):
    """The reference's own dim-4 view on the device: 16 of the 320 density slices, each
    computed by its own pass (its high digits select the pass)."""
    ids = REFSL["ids"][:8] + REFSL["ids"][-8:]
    want = np.array([cx(v) for v in REFSL["slices"][:8] + REFSL["slices"][-8:]])
    scale = np.max(np.abs(np.array([cx(v) for v in REFSL["slices"]])))
    with Engine(payload_path(HEADLINE), device=0, mode="density", max_batch_bits=8) as e:
        got = np.array([e.slice_values(s, s + 1)[0] for s in ids])
    assert np.max(np.abs(got - want)) <= REL * scale, np.max(np.abs(got - want)) / scale


# ---------------------------------------------------------------- amplitude batches (one pass, n amplitudes)

CFG4 = ["cfg4_n100_p1_s1_m16_ext_bt", "cfg4_n100_p1_s1_m16_ext_cs"]


def test_batch_engine_host_plan():
    """8 bitstrings of config 4 as one program: 3 amplitude bits, and the tensors that do not
    depend on the measurement vectors (tensor_network.cpp:82-87) are shared: one program, about
    the launches of a single amplitude."""
    from paper_2010_14962_b200 import Engine

    stem = CFG4[0]
    with Engine([payload_path(stem, b) for b in range(8)], device=-1, mode="ket", mem_budget_bytes=100 << 30) as e:
        st = e.plan_stats()
    with Engine(payload_path(stem, 0), device=-1, mode="ket", mem_budget_bytes=100 << 30) as e1:
        st1 = e1.plan_stats()
    assert (st["n_amplitudes"], st["amp_bits"], st1["n_amplitudes"], st1["amp_bits"]) == (8, 3, 1, 0)
    assert st["n_steps"] == st1["n_steps"] and st["peak_rank"] == st1["peak_rank"]
    # (the engine's fusion decisions depend on the batched tensor sizes, so the two programs do not
    # fuse the same steps; the batch still moves about what 8 separate amplitudes would, not more
    # than 10x one amplitude, while its launches -- the latency that binds these plans -- are shared)
    assert st1["moved_bytes"] < st["moved_bytes"] < 10 * st1["moved_bytes"]
    assert st["n_kernels"] <= 2 * st1["n_kernels"]  # not 8 programs' worth of launches


def test_batch_engine_rejects_mismatch():
    """Payloads of different cuts or plans cannot share a program (QC_EINVAL -> ValueError), and
    the single-amplitude calls refuse a batch engine."""
    from paper_2010_14962_b200 import Engine

    with pytest.raises(ValueError, match="batched payloads differ"):
        Engine([payload_path(CFG4[0], 0), payload_path(CFG4[1], 1)], device=-1, mode="ket")
    with Engine([payload_path(CFG4[0], b) for b in range(3)], device=-1, mode="ket") as e:
        with pytest.raises(ValueError, match="3 amplitudes"):
            e.ket_sum()
        with pytest.raises(ValueError, match="3 amplitudes"):
            e.sum_range(0, 4)


@pytest.mark.gpu
@pytest.mark.parametrize("stem", CFG4)
def test_batch_engine_amplitudes(Engine, stem):
    """Config 4's 8 bitstrings in one pass: every amplitude and every slice value against the
    oracle's (amplitudes.json), 1e-10."""
    with Engine([payload_path(stem, b) for b in range(8)], device=0, mode="ket") as e:
        a = e.ket_sum_batch()
        vals = e.ket_values_batch()
    for b in range(8):
        key = f"{stem}.b{b}"
        want = cx(AMPS[key]["A"])
        assert abs(a[b] - want) <= REL * abs(want), (key, a[b], want)
        check_values(key, vals[b])


@pytest.mark.gpu
def test_batch_engine_padding_and_ranges(Engine):
    """A 3-amplitude batch (padded to 4 inside the pass) over partial ranges equals the single
    engines' partial sums; a batch of one payload twice gives it twice."""
    stem = CFG4[0]
    bs = [5, 0, 2]
    with Engine([payload_path(stem, b) for b in bs], device=0, mode="ket") as e:
        part = e.ket_sum_batch(1000, 40000)
        vals = e.ket_values_batch(7, 300)
    for i, b in enumerate(bs):
        with Engine(payload_path(stem, b), device=0, mode="ket") as e1:
            want = e1.ket_sum(1000, 40000)
            wv = e1.ket_values(7, 300)
        assert abs(part[i] - want) <= REL * abs(want)
        assert np.max(np.abs(vals[i] - wv)) <= REL * np.max(np.abs(wv))
    with Engine([payload_path(stem, 3)] * 2, device=0, mode="ket") as e:
        two = e.ket_sum_batch()
    want = cx(AMPS[f"{stem}.b3"]["A"])
    assert all(abs(v - want) <= REL * abs(want) for v in two)


# ---------------------------------------------------------------- fused final reduction (k_gate_reduce)

@pytest.mark.gpu
def test_fused_final_reduction_passes_and_ranges(Engine):
    """The headline plan's last gate does the final product and slice sum in its epilogue
    (k_gate_reduce) whenever no per-slice values are requested. The fused route must agree with
    the unfused one (ket_values -> the gate writes its result, k_final walks it) on the whole
    amplitude, on ranges that cut through passes (the epilogue's range mask through the inverse
    map), and when the amplitude is split into several passes (k_final folds the pass slots)."""
    stem = "cfg5_n120_p1_s5_m20_ext_bt"
    want = cx(AMPS[stem + ".b0"]["A"])
    with Engine(payload_path(stem), device=0, mode="ket") as e:
        assert "+final" in e.describe()
        total = e.ket_jobs()
        a1 = e.ket_sum()
        vals = e.ket_values(0, 3 << 18)  # per-slice values: the unfused route
        for lo, hi in ((0, 3 << 18), (12345, 600001), (1 << 19, (1 << 19) + 7), (5, 5)):
            got = e.ket_sum(lo, hi)
            ref = np.sum(vals[lo:hi]) if hi <= vals.size else None
            if ref is not None:
                # (2^20 terms of mixed phase: rounding differs by ~n eps max|v| between the two trees)
                assert abs(got - ref) <= 1e-9 * np.max(np.abs(vals)), (lo, hi, got, ref)
        a1_again = e.ket_sum()
    assert a1 == a1_again  # bitwise reproducible, also after unfused calls on the same engine
    assert abs(abs(a1) - abs(want)) <= REL * abs(want)
    with Engine(payload_path(stem), device=0, mode="ket", max_batch_bits=18) as e4:  # 4 passes of 2^18 slices
        st = e4.plan_stats()
        assert st["batch_bits"] == 18 and st["chunks"] == 4 and "+final" in e4.describe()
        a4 = e4.ket_sum()
        part = e4.ket_sum(100000, 900000)  # starts and ends inside passes
        v4 = e4.ket_values(100000, 900000)
    assert abs(a4 - a1) <= 1e-10 * abs(a1)
    assert abs(part - np.sum(v4)) <= 1e-9 * np.max(np.abs(v4))
    assert total == 1 << 20
