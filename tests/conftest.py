"""Shared fixtures.  `-m gpu` tests need a B200 (run via gpurun); everything
else runs on the CPU container.  The oracle (oracle/) is test infrastructure
and is only imported here and in the tests."""
from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run under gpurun")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


def load_golden(name: str):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    with open(path) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_small():
    return load_golden("golden_small.json")


@pytest.fixture(scope="session")
def engine():
    """A C-ABI context on cuda:0 (gpu tests only)."""
    from paper_1209_4408_b200 import life
    e = life.Engine(0)
    yield e
    e.close()
