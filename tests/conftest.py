"""Test configuration.

* ``gpu`` marks tests that launch kernels on a B200 (run by the driver with
  ``-m gpu``); everything else must pass on a GPU-less host.
* Every test gets a fresh runtime (mirrors the reference fixture
  tests/conftest.py:6-10).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import _native  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def pytest_collection_modifyitems(config, items):
    if _native.device_count() > 0:
        return
    skip = pytest.mark.skip(reason="no CUDA device available")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(autouse=True)
def fresh_runtime():
    sf.init_runtime(sf.RuntimeOptions())
    yield


@pytest.fixture
def host_rng_runtime():
    """Parity mode: random draws come from the reference's PCG64 stream."""
    return sf.init_runtime(sf.RuntimeOptions(rng="host"))
