import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU")
    config.addinivalue_line("markers", "slow: long-running (large images)")


@pytest.fixture(scope="session")
def small_cases():
    z = np.load(os.path.join(GOLDEN, "small_cases.npz"))
    names = sorted(k[len("img__"):] for k in z.files if k.startswith("img__"))
    return {n: (z["img__" + n], z["lab__" + n]) for n in names}


@pytest.fixture(scope="session")
def known_answers():
    import json
    with open(os.path.join(GOLDEN, "known_answers.json")) as f:
        return {d["name"]: d for d in json.load(f)["answers"]}


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def ccl():
    import paper_1712_09789_b200 as ccl
    return ccl
