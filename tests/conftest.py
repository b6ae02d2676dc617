import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden", "reference_golden.json")
CANON_INIT = ("-15.8", "-17.48", "35.64")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as fh:
        data = json.load(fh)
    return {c["name"]: c for c in data["cases"]}


@pytest.fixture(scope="session")
def gpu():
    """The CUDA engine; GPU tests fail (not skip) when it cannot load."""
    from paper_1908_09301_b200 import _native

    return _native.load()
