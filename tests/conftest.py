import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity via the C-ABI")


@pytest.fixture(scope="session")
def known():
    with open(os.path.join(GOLDEN, "known.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def configs():
    with open(os.path.join(GOLDEN, "configs.json")) as f:
        return json.load(f)


def load_small():
    z = np.load(os.path.join(GOLDEN, "small.npz"))
    cases = {}
    for k in z.files:
        name, field = k.split("/", 1)
        cases.setdefault(name, {})[field] = z[k]
    return cases


SMALL = load_small()
SMALL_NAMES = sorted(SMALL)


@pytest.fixture(scope="session")
def small():
    return SMALL
