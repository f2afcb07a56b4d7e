"""Shared fixtures.  `-m "not gpu"` runs here (no GPU): oracle vs golden
vectors, host logic, C-ABI exports.  `-m gpu` runs on a B200: parity of the
CUDA path (through the C ABI) against the oracle and the golden vectors."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def g_tables():
    from _hb_util import golden

    return golden("tables")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.build()
    return O
