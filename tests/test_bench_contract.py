"""bench.py's output contract: the reference arm (CPU, runs here) and the engine arm (GPU).

The reference arm times the UNMODIFIED reference's sum_range on the host cores
(oracle/_ref/qcut_refgen bench -> qcut::sum_range on run_pool's grid) for the same metric,
unit and config as the engine arm, and says what it sampled and what it extrapolated.
"""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e")


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "qcut_refgen")),
                    reason="the compiled reference (oracle/_ref) is built where /root/reference exists")
def test_reference_arm_line_config1():
    """BASELINE config 1 fits the reference's CPU path whole: full amplitudes are timed, nothing
    is extrapolated, and the line carries the engine arm's metric, unit and config keys."""
    d = run_bench("--impl", "reference", "--config", "cfg1", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference"
    for k in KEYS:
        assert k in d, k
    assert d["metric"] == "slices/s" and d["unit"] == "slices/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert "full amplitudes" in d["cpu_baseline"]["sample"]
    assert d["cpu_baseline"]["value"] == d["value"] == d["e2e"]["value"] and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["ms_per_step"] > 0 and d["like_for_like_port"]["kind"] == "port"
    assert d["config"]["k"] == 4 and "config 1" in d["config"]["workload"]


@pytest.mark.gpu
def test_engine_arm_line_default():
    """The default bench line (BASELINE config 5) carries the contract's keys, the roofline of the
    time-dominant launch, the pass-level roofline, clocks, e2e with the host copies declared,
    the launch count and the amplitude, which must be the oracle's."""
    d = run_bench("--steps", "3", "--warmup", "3", "--cpu-seconds", "2")
    for k in KEYS + ("roofline", "pass_roofline", "clocks", "gpu_launches", "amplitude"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["dtype"] == "complex128" and d["vs_baseline"] is None
    assert "config 5" in d["config"]["workload"] and d["config"]["slices_per_step"] == 1 << 20
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "kernel"):
        assert k in r, k
    assert abs(r["frac"] - r["achieved"] / r["peak"]) <= 1e-9
    assert 0 < d["pass_roofline"]["hbm_frac"] <= 1.2 and 0 < d["pass_roofline"]["fp64_frac"] <= 1.2
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] == 16
    assert d["e2e"]["value"] < d["value"] and d["gpu_launches"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] > 0
    with open(os.path.join(ROOT, "tests", "golden", "amplitudes.json")) as f:
        want = json.load(f)["cfg5_n120_p1_s5_m20_ext_bt.b0"]["abs2"]
    assert abs(d["amplitude"]["abs2"] - want) <= 1e-10 * want
