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


def record_parity(what, rel_l2, max_over_rms, max_over_max=None):
    """Append one achieved parity margin to $GBS_PARITY_LOG (JSON lines), if set."""
    path = os.environ.get("GBS_PARITY_LOG")
    if not path:
        return
    with open(path, "a") as f:
        f.write(json.dumps({"case": what, "rel_l2": rel_l2, "max_abs_over_rms": max_over_rms,
                            "max_abs_over_max": max_over_max}) + "\n")
