"""Parity of the sm_100a engine (through the C-ABI) against the reference and the oracle.

Tolerances: complex128 results within 1e-10 relative of the reference (BASELINE
north star); per-slice values within 1e-10 of the largest slice magnitude.
Bit-exact items: per-step shapes, slice enumeration (slice ids and count).
"""
import numpy as np
import pytest

from conftest import RANDOM_STEMS, SMALL_QAOA, cx, payload_path, ref_json

pytestmark = pytest.mark.gpu

REL = 1e-10


@pytest.fixture(scope="module")
def Engine():
    from paper_2010_14962_b200 import Engine as E

    return E


def close(a, b, rel=REL, floor=0.0):
    return abs(a - b) <= rel * max(abs(b), floor) + 1e-300


def dephase(a, ref):
    """Remove the single global phase of the ket view (fixed by the factorisation convention)."""
    c = np.vdot(a, ref)
    return a * (c / abs(c)) if abs(c) > 0 else a


@pytest.mark.parametrize("stem", SMALL_QAOA + ["n10_p2_s1_m4", "cnot", "flip"] + RANDOM_STEMS)
def test_density_view_matches_reference(Engine, stem):
    ref = ref_json(stem)
    want = cx(ref.get("run_serial", ref.get("run_pool8", ref.get("serial"))))
    with Engine(payload_path(stem), device=0, mode="density") as e:
        got = e.run_serial()
        assert close(got, want, floor=1e-12), (got, want)
        if "slices" in ref:
            sl = np.array([cx(v) for v in ref["slices"]])
            vals = e.slice_values(0, e.jobs())
            assert np.max(np.abs(vals - sl)) <= REL * max(1e-12, np.max(np.abs(sl)))


@pytest.mark.parametrize("stem", SMALL_QAOA + ["n10_p2_s1_m4"] + RANDOM_STEMS)
def test_ket_view_matches_reference(Engine, oracle_mod, stem):
    ref = ref_json(stem)
    want = cx(ref.get("run_serial", ref.get("run_pool8", ref.get("serial"))))
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path(stem)), "ket")
    _, ka = net.sum_range(0, net.jobs, per_slice=True)
    with Engine(payload_path(stem), device=0, mode="ket") as e:
        p = e.run_serial()
        assert close(p, want, floor=1e-12), (p, want)
        vals = e.ket_values()
        assert np.max(np.abs(dephase(vals, ka) - ka)) <= REL * max(1e-12, np.max(np.abs(ka)))
        if "slices" in ref:  # density-id per-slice values answered from the ket view
            sl = np.array([cx(v) for v in ref["slices"]])
            assert np.max(np.abs(e.slice_values(0, e.jobs()) - sl)) <= REL * max(1e-12, np.max(np.abs(sl)))


@pytest.mark.parametrize("mode", ["density", "ket"])
def test_partial_ranges_and_additivity(Engine, mode):
    """sum_range over arbitrary [lo, hi) == sum of the reference per-slice values (test_executor.cpp:92-99)."""
    ref = ref_json("cfg1_n20_p1_s1_m4")
    sl = np.array([cx(v) for v in ref["slices"]])
    with Engine(payload_path("cfg1_n20_p1_s1_m4"), device=0, mode=mode) as e:
        for lo, hi in [(0, 1), (3, 4), (0, 100), (100, 256), (17, 211), (255, 256), (5, 5), (64, 128)]:
            got = e.sum_range(lo, hi)
            want = sl[lo:hi].sum()
            assert abs(got - want) <= REL * max(1e-12, np.abs(sl).max()) * max(1, hi - lo), (lo, hi)
        whole = e.sum_range(0, 256)
        assert abs(whole - (e.sum_range(0, 77) + e.sum_range(77, 256))) <= 1e-12 * abs(whole)


def test_small_batches_and_passes_agree(Engine, oracle_mod):
    """Forcing a small memory budget splits the range into many device passes; results must not change."""
    stem = "n24_p1_s1_m5"
    ref = ref_json(stem)
    sl = np.array([cx(v) for v in ref["slices"]])
    for mode in ("density", "ket"):
        # one byte less than the single-pass workspace forces a multi-pass program
        with Engine(payload_path(stem), device=-1, mode=mode, mem_budget_bytes=1 << 40) as h:
            budget = h.plan_stats()["arena_bytes"] - 1
        with Engine(payload_path(stem), device=0, mode=mode, mem_budget_bytes=budget) as e:
            st = e.plan_stats()
            assert st["chunks"] > 1
            assert close(e.run_serial(), cx(ref["run_serial"]))
            assert np.max(np.abs(e.slice_values(100, 400) - sl[100:400])) <= REL * np.abs(sl).max()


def test_bitwise_reproducible(Engine):
    with Engine(payload_path("cfg2_n60_p1_s1_m10_ext"), device=0, mode="ket") as e:
        a = e.ket_sum()
        b = e.ket_sum()
        assert a == b


def test_errors_map_to_reference_exceptions(Engine):
    from paper_2010_14962_b200 import RankGuardError

    with Engine(payload_path("cfg1_n20_p1_s1_m4"), device=0, mode="ket") as e:
        with pytest.raises(ValueError, match="outside"):
            e.sum_range(2, 1)
        with pytest.raises(ValueError, match="outside"):
            e.sum_range(0, 257)
    import gzip
    import json

    with gzip.open(payload_path("cfg1_n20_p1_s1_m4"), "rt") as f:
        p = json.load(f)
    p["max_rank"] = 3
    with Engine(json.dumps(p).encode(), device=0, mode="ket") as e:
        with pytest.raises(RankGuardError) as ei:
            e.run_serial()
        assert ei.value.max_rank == 3 and ei.value.rank > 3


def test_config2_ket_amplitude_vs_oracle(Engine, oracle_mod):
    """BASELINE config 2 (N=60, k=10, peak 16): the reference CPU path cannot run it (dim-4 peak 16);
    the ket-view oracle port can. |A|^2 and every ket slice value must agree to 1e-10."""
    stem = "cfg2_n60_p1_s1_m10_ext"
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path(stem)), "ket")
    a_ref, ka = net.sum_range(0, net.jobs, per_slice=True)
    with Engine(payload_path(stem), device=0, mode="ket") as e:
        assert e.plan_stats()["peak_rank"] == 16
        a = e.ket_sum()
        assert abs(abs(a) - abs(a_ref)) <= REL * abs(a_ref)
        vals = e.ket_values()
        assert np.max(np.abs(dephase(vals, ka) - ka)) <= REL * np.abs(ka).max()
        assert close(e.run_serial().real, abs(a_ref) ** 2)


def test_config2_default_plan_peak21(Engine, oracle_mod):
    """Config 2 with the default GA budget (peak 21, ~38 GB workspace at full batch)."""
    stem = "cfg2_n60_p1_s1_m10"
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path(stem)), "ket")
    a_ref, ka = net.sum_range(0, 8, per_slice=True)
    with Engine(payload_path(stem), device=0, mode="ket") as e:
        vals = e.ket_values(0, 8)
        assert np.max(np.abs(dephase(vals, ka) - ka)) <= REL * np.abs(ka).max()


def test_config4_sampled_slices_vs_oracle(Engine, oracle_mod):
    """Config 4 (N=100, k=16, peak 22): ket slices sampled against the oracle port, and the
    full amplitude is invariant to the pass decomposition."""
    stem = "cfg4_n100_p1_s1_m16_ext"
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path(stem)), "ket")
    _, ka = net.sum_range(0, 2, per_slice=True)
    with Engine(payload_path(stem), device=0, mode="ket") as e:
        assert e.plan_stats()["peak_rank"] == 22
        vals = e.ket_values(0, 2)
        assert np.max(np.abs(dephase(vals, ka) - ka)) <= REL * np.abs(ka).max()
        full = e.ket_sum()
        halves = e.ket_sum(0, 1 << 15) + e.ket_sum(1 << 15, 1 << 16)
        assert abs(full - halves) <= 1e-9 * abs(full)


def test_step_shapes_match_reference_plan(Engine):
    import gzip
    import json

    for stem in ["cfg1_n20_p1_s1_m4", "cfg2_n60_p1_s1_m10_ext"]:
        with gzip.open(payload_path(stem), "rt") as f:
            steps = json.load(f)["plan"]["steps"]
        want = np.array([[s["rank_a"], s["rank_b"], len(s["edges"]), s["result_rank"]] for s in steps])
        for mode in ("ket", "density"):
            with Engine(payload_path(stem), device=0 if stem.startswith("cfg1") else -1, mode=mode) as e:
                assert np.array_equal(e.step_shapes(), want)


def test_reference_side_shim():
    """include/qcut_gpu_shim.hpp compiled against the unmodified reference library
    (oracle/_ref/shim_demo): reference run_serial (CPU) == engine via the shim, a
    run_pool-grid pool over eng.sum_range + reference aggregate, RankGuardError mapping."""
    import os
    import subprocess
    import tempfile
    import gzip

    from conftest import ROOT

    exe = os.path.join(ROOT, "oracle", "_ref", "shim_demo")
    assert os.path.exists(exe), "shim_demo not built (build() compiles it where /root/reference exists)"
    for stem in ("cfg1_n20_p1_s1_m4", "random_n4_d10_s7_m3"):
        with tempfile.NamedTemporaryFile(suffix=".json", delete=False) as tf, gzip.open(payload_path(stem)) as g:
            tf.write(g.read())
        for mode in ("0", "1"):
            r = subprocess.run([exe, tf.name, mode], capture_output=True, text=True, timeout=300)
            assert r.returncode == 0, r.stdout + r.stderr
        os.unlink(tf.name)


def test_reference_file_inputs_through_shim():
    """the reference's own circuit and cut files (emit_circuit / dump_cut_json,
    tests/golden/*.circuit, *.cut.json) -> qcut::gpu::job_from_files (graph-hash check as
    tools/qcut.cpp:69-78, make_job as `qcut run`) -> engine; equals the reference run_serial
    of the same JobSpec and the golden value; a cut file for another network is refused."""
    import json
    import os
    import subprocess

    from conftest import ROOT, golden

    exe = os.path.join(ROOT, "oracle", "_ref", "shim_demo")
    assert os.path.exists(exe), "shim_demo not built (build() compiles it where /root/reference exists)"
    for stem, other in (("cfg1_n20_p1_s1_m4", "readme_n12_s7_m2"), ("readme_n12_s7_m2", "cfg1_n20_p1_s1_m4")):
        for mode in ("0", "1"):
            r = subprocess.run([exe, "--files", golden(stem + ".b0.circuit"), golden(stem + ".cut.json"),
                                golden(other + ".b0.circuit"), mode], capture_output=True, text=True, timeout=300)
            assert r.returncode == 0, r.stdout + r.stderr
            out = json.loads(r.stdout.strip().splitlines()[-1])
            assert close(cx(out["gpu"]), cx(ref_json(stem)["run_serial"]), floor=1e-12)


def test_capped_batch_matches_uncapped(Engine):
    """Per-rank engines of a sharded run (max_batch_bits = log2 of the shard) give the same
    shard sums as the single full-batch engine."""
    stem = "cfg2_n60_p1_s1_m10_ext"
    with Engine(payload_path(stem), device=0, mode="ket") as e:
        full = [e.ket_sum(g * 256, (g + 1) * 256) for g in range(4)]
    for g in range(4):
        with Engine(payload_path(stem), device=0, mode="ket", max_batch_bits=8) as e:
            assert e.plan_stats()["batch_bits"] == 8
            got = e.ket_sum(g * 256, (g + 1) * 256)
            assert abs(got - full[g]) <= REL * max(abs(full[g]), 1e-30) + 1e-25


def test_long_call_runs_in_pass_chunks(Engine):
    """A call spanning more passes than the pass buffers hold (2^14) runs in chunks of
    whole passes folded in order: same density-range sum as a full-batch engine, and the
    per-slice values of a window across a chunk boundary agree (config 2, searched cut,
    density view, one density slice per pass)."""
    stem = "cfg2_n60_p1_s1_m10_ext_cs"
    lo, hi = 3000, 3000 + (1 << 14) + 700
    with Engine(payload_path(stem), device=0, mode="density") as e:
        want = e.sum_range(lo, hi)
        wper = e.slice_values(lo + (1 << 14) - 8, lo + (1 << 14) + 8)
    with Engine(payload_path(stem), device=0, mode="density", max_batch_bits=0) as e:
        assert e.plan_stats()["batch_bits"] == 0
        got = e.sum_range(lo, hi)
        gper = e.slice_values(lo + (1 << 14) - 8, lo + (1 << 14) + 8)
        assert e.last_run()["launches"] > 0
    scale = max(abs(want), np.abs(wper).max(), 1e-300)
    assert abs(got - want) <= REL * scale * 100, (got, want)
    assert np.max(np.abs(gper - wper)) <= REL * np.abs(wper).max()


@pytest.mark.gpu
def test_contract_pair_through_the_cpp_shim():
    """qcut::gpu::contract_pair (include/qcut_gpu_shim.hpp) against the unmodified reference's
    qcut::contract_pair, both called from C++ (oracle/_ref/shim_demo --pair): BM_ContractPair's
    shapes, a mixed leg order, and the exception mapping."""
    import json
    import os
    import subprocess

    from conftest import ROOT

    exe = os.path.join(ROOT, "oracle", "_ref", "shim_demo")
    assert os.path.exists(exe), "shim_demo not built (build() compiles it where /root/reference exists)"
    r = subprocess.run([exe, "--pair"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["worst_rel"] <= 1e-12 and out["invalid_argument"] and out["rank_guard"]
