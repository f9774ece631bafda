"""Shared pytest setup: the `gpu` marker, golden fixtures, and path wiring.

CPU tests (`-m "not gpu"`) cover the oracle against the golden vectors, the
host-side logic and the C-ABI exports; `-m gpu` tests run the CUDA path on a
B200 and compare it with the oracle.
"""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return GOLDEN


@pytest.fixture
def rng():
    return np.random.default_rng(2024)
