"""C-ABI library: loads, exports every declared symbol, host-side planning and
error mapping (no compute calls; runs without a GPU)."""
import gzip
import json
import os
import re

import numpy as np
import pytest

from conftest import ALL_PAYLOAD_STEMS, ROOT, payload_path, ref_json


def header_symbols():
    with open(os.path.join(ROOT, "include", "qcut_gpu.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"QC_API\s+[\w\s\*]+?\b(qc_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2010_14962_b200.engine import EXPORTS, load_library

    lib = load_library()
    syms = header_symbols()
    assert len(syms) >= 12
    assert sorted(EXPORTS) == syms
    for s in syms:
        assert hasattr(lib, s), s
    assert b"sm_100a" in lib.qc_version()


@pytest.mark.parametrize("stem", ALL_PAYLOAD_STEMS)
def test_host_plan_shapes_match_reference(stem):
    """Intermediate shapes are bit-exact with the reference plan in both views."""
    from paper_2010_14962_b200 import Engine

    with gzip.open(payload_path(stem), "rt") as f:
        p = json.load(f)
    want = np.array([[s["rank_a"], s["rank_b"], len(s["edges"]), s["result_rank"]] for s in p["plan"]["steps"]])
    for mode in ("ket", "density"):
        if mode == "density" and p["plan"]["peak_rank"] > 12:
            continue  # density view of configs 2-5 is the infeasible reference formulation
        with Engine(payload_path(stem), device=-1, mode=mode) as e:
            st = e.plan_stats()
            assert st["n_steps"] == len(p["plan"]["steps"])
            assert st["peak_rank"] == p["plan"]["peak_rank"]
            assert st["jobs"] == 4 ** len(p["cut"])
            assert np.array_equal(e.step_shapes().reshape(-1, 4), want.reshape(-1, 4))


def _payload():
    with gzip.open(payload_path("cfg1_n20_p1_s1_m4"), "rt") as f:
        return json.load(f)


def test_errors_without_device():
    from paper_2010_14962_b200 import Engine, RankGuardError

    p = _payload()
    with pytest.raises(ValueError, match="json"):
        Engine(b"{not json", device=-1)
    bad = json.loads(json.dumps(p))
    bad["cut"] = list(reversed(bad["cut"]))
    with pytest.raises(ValueError, match="sorted"):
        Engine(json.dumps(bad).encode(), device=-1)
    bad = json.loads(json.dumps(p))
    bad["cut"] = [bad["cut"][0], bad["cut"][0]]
    with pytest.raises(ValueError, match="repeats"):
        Engine(json.dumps(bad).encode(), device=-1)
    bad = json.loads(json.dumps(p))
    bad["plan"]["steps"][3]["legs_a"] = [9]
    with pytest.raises(ValueError, match="out of range"):
        Engine(json.dumps(bad).encode(), device=-1)
    bad = json.loads(json.dumps(p))
    bad["network"]["edges"].pop()
    with pytest.raises(ValueError, match="not closed"):
        Engine(json.dumps(bad).encode(), device=-1)
    bad = json.loads(json.dumps(p))
    del bad["plan"]["steps"][-1]
    with pytest.raises(ValueError, match="scalar"):
        Engine(json.dumps(bad).encode(), device=-1)
    # rank guard: raised by the compute call, like sum_range (executor.cpp:53)
    guarded = json.loads(json.dumps(p))
    guarded["max_rank"] = 3
    with Engine(json.dumps(guarded).encode(), device=-1) as e:
        with pytest.raises(RankGuardError) as ei:
            e.run_serial()
        first = next(s["result_rank"] for s in p["plan"]["steps"] if s["result_rank"] > 3)
        assert ei.value.rank == first and ei.value.max_rank == 3
        assert f"rank-{first} tensor ({16.0 * 4 ** first:.6f} bytes), exceeding max rank 3" in str(ei.value)
    with Engine(payload_path("cfg1_n20_p1_s1_m4"), device=-1) as e:
        with pytest.raises(ValueError, match=r"range \[2,1\) outside \[0,256\)"):
            e.sum_range(2, 1)
        with pytest.raises(RuntimeError, match="without a device"):
            e.sum_range(0, 1)


def test_ket_view_rejects_mixed_inputs():
    """The ket view needs T = K (x) conj(K); a mixed input state must be refused (EINVAL)."""
    from paper_2010_14962_b200 import Engine

    p = _payload()
    for v in p["network"]["vertices"]:
        if v["id"] == 0:
            v["data"] = [[0.5, 0.0], [0.0, 0.0], [0.0, 0.0], [0.5, 0.0]]
    with pytest.raises(ValueError, match="factorise"):
        Engine(json.dumps(p).encode(), device=-1, mode="ket")
    with Engine(json.dumps(p).encode(), device=-1, mode="density") as e:
        assert e.plan_stats()["n_steps"] == len(p["plan"]["steps"])


def test_accounting_matches_survey_definition():
    """essential bytes = sum over slice-dependent steps of 16 (2^ra + 2^rb + 2^rr) x slices + invariant once."""
    from paper_2010_14962_b200 import Engine

    p = json.load(gzip.open(payload_path("cfg2_n60_p1_s1_m10_ext"), "rt"))
    with Engine(payload_path("cfg2_n60_p1_s1_m10_ext"), device=-1, mode="ket") as e:
        st = e.plan_stats()
    # SURVEY §8(d) quotes 3.38e6 B per slice for this plan; x 1024 slices ~ 3.4e9 (+ invariant steps)
    assert 3.3e9 < st["essential_bytes"] < 3.5e9
    assert st["moved_bytes"] <= st["essential_bytes"]
    assert st["n_invariant_steps"] > 0.6 * len(p["plan"]["steps"])


@pytest.mark.parametrize("stem", ALL_PAYLOAD_STEMS)
def test_program_validation_over_batch_choices(stem):
    """compute-sanitizer is closed on the GPU pool, so every device program is validated on the
    host at build time (program.cpp: every index map's largest value inside its tensor, every
    tensor inside the workspace, no two simultaneously-live tensors aliased). Exercise it over
    single-pass and many-pass programs of every golden payload in both views."""
    from paper_2010_14962_b200 import Engine

    with gzip.open(payload_path(stem), "rt") as f:
        peak = json.load(f)["plan"]["peak_rank"]
    for mode in ("ket", "density"):
        if mode == "density" and peak > 10:
            continue
        with Engine(payload_path(stem), device=-1, mode=mode, mem_budget_bytes=1 << 44) as e:
            full = e.plan_stats()["arena_bytes"]
        for budget in (full, full - 1, full // 4, full // 64):
            try:
                with Engine(payload_path(stem), device=-1, mode=mode, mem_budget_bytes=budget) as e:
                    st = e.plan_stats()
                    assert st["arena_bytes"] <= budget
            except RuntimeError as ex:  # a single slice does not fit: reported, never a bad program
                assert "exceeds the memory budget" in str(ex)


@pytest.mark.parametrize("stem", ["cfg1_n20_p1_s1_m4", "readme_n12_s7_m2"])
def test_reference_file_inputs_host_only(stem):
    """The reference's circuit + cut files through qcut::gpu::job_from_files (shim) into a
    host-only engine (device -1): plan statistics agree with the JobSpec, and a cut file
    built for another network fails the graph-hash check (tools/qcut.cpp:69-78)."""
    import subprocess

    from conftest import ROOT, golden

    exe = os.path.join(ROOT, "oracle", "_ref", "shim_demo")
    if not os.path.exists(exe):
        pytest.skip("shim_demo needs the reference build (oracle/Makefile)")
    other = "readme_n12_s7_m2" if stem.startswith("cfg1") else "cfg1_n20_p1_s1_m4"
    r = subprocess.run([exe, "--check-files", golden(stem + ".b0.circuit"), golden(stem + ".cut.json"),
                        golden(other + ".b0.circuit")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["hash_check"] is True
    assert out["jobs"] == 4 ** len(ref_json(stem)["info"]["cut"])


def test_max_batch_bits_caps_the_pass():
    """qc_engine_create_ex: a sharded caller caps the batched slice bits at its shard size
    (bench.py for --gpus N), so a pass never computes other ranks' slices."""
    from paper_2010_14962_b200 import Engine

    for cap in (0, 3, 7, 10):
        with Engine(payload_path("cfg2_n60_p1_s1_m10_ext"), device=-1, mode="ket", max_batch_bits=cap) as e:
            st = e.plan_stats()
            assert st["batch_bits"] == min(cap, 10) and st["chunks"] == 2 ** (10 - min(cap, 10))
