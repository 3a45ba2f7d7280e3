import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        meta = json.load(fh)
    arrays = dict(np.load(os.path.join(GOLDEN, "golden.npz")))
    return meta, arrays


@pytest.fixture(scope="session")
def gpu():
    from paper_2406_14084_b200 import _lib
    _lib.lib()  # a missing library is an error, never a skip
    if _lib.device_count() < 1:
        pytest.skip("no CUDA device in this container")
    return True


# reference worked example (pkg/tests/conftest.py:8-56)
EXAMPLE_RAW = """H 0 0
H 1 1
RZZ 2 4 2
RZZ 5 7 3
H 8 4
H 9 5
H 3 6
H 6 7
RZZ 0 2 8
RZZ 4 7 9
H 9 10
RZZ 1 8 11
RZZ 3 6 12
H 5 13
"""

from __graft_entry__ import _EXAMPLE as EXAMPLE_OPTIMIZED  # noqa: E402,F401
