"""Shared fixtures and markers.

`-m "not gpu"` runs here (no GPU): oracle-vs-golden pins, host logic, the
C-ABI library's exports, multi-rank host logic over gloo.
`-m gpu` runs on a B200: CUDA path vs the oracle and the golden fixtures.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]

    return get


@pytest.fixture(scope="session")
def ns():
    from paper_2308_01651_b200 import configs

    return configs.this_package()
