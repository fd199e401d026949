import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def paper():
    with open(os.path.join(GOLDEN, "paper_values.json")) as f:
        return json.load(f)


@pytest.fixture(autouse=True, scope="session")
def _oracle_threads():
    try:
        from oracle import c_oracle
        c_oracle.set_threads(os.cpu_count() or 1)
    except Exception:
        pass
    yield
