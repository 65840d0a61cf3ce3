import glob
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden(name: str) -> str:
    return os.path.join(GOLD, name)


def ref_json(stem: str) -> dict:
    with open(golden(stem + ".ref.json")) as f:
        return json.load(f)


def payload_path(stem: str, b: int = 0) -> str:
    p = golden(f"{stem}.b{b}.payload.json.gz")
    return p if os.path.exists(p) else golden(f"{stem}.payload.json.gz")


def cx(v) -> complex:
    return complex(v[0], v[1])


RANDOM_STEMS = sorted(os.path.basename(p)[: -len(".ref.json")] for p in glob.glob(os.path.join(GOLD, "random_*.ref.json")))
SMALL_QAOA = ["cfg1_n20_p1_s1_m4", "readme_n12_s7_m2", "n24_p1_s1_m5"]
ALL_PAYLOAD_STEMS = SMALL_QAOA + ["n10_p2_s1_m4", "cnot", "flip", "cfg2_n60_p1_s1_m10_ext", "cfg2_n60_p1_s1_m10",
                                  "cfg4_n100_p1_s1_m16_ext", "cfg5_n120_p1_s5_m20_ext", "cfg2_n60_p1_s1_m10_ext_os",
                                  "cfg4_n100_p1_s1_m16_ext_os", "cfg5_n120_p1_s5_m20_ext_os", "cfg1_n20_p1_s1_m4_split",
                                  "cfg2_n60_p1_s1_m10_ext_split"] + RANDOM_STEMS


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O

    if not os.path.exists(O.LIB_PATH):
        O.build(ref=False)
    return O
