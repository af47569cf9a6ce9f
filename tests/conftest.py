"""Shared pytest setup.

Markers: `gpu` -- needs a CUDA device (run on the B200 box with -m gpu);
everything unmarked runs on CPU in the build container.
"""

import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")

P1, P2, P3 = 469762049, 998244353, 2013265921


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_small():
    with open(os.path.join(GOLDEN, "reference_small.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_configs():
    with open(os.path.join(GOLDEN, "reference_configs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle

    oracle.lib()
    return oracle
