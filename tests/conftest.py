import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)

from peeltest_util import load_goldens, load_oracle_goldens  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-scale) case")




@pytest.fixture(scope="session")
def goldens():
    """SURVEY §8 c3's independent goldens: used by the oracle pins (-m "not gpu")."""
    return load_goldens()


@pytest.fixture(scope="session")
def oracle_goldens():
    """tools/make_oracle_goldens.py's oracle-computed values: the GPU tests' expected values."""
    return load_oracle_goldens()
