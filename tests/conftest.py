"""Test configuration: the `gpu` marker and import paths.

`-m "not gpu"` runs on any CPU box (oracle vs golden fixtures, host logic,
C-ABI exports); `-m gpu` needs a B200 and calls the CUDA path through the
C-ABI library.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
