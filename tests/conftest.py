import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np
    arrays = dict(np.load(os.path.join(GOLDEN, "golden_small.npz")))
    with open(os.path.join(GOLDEN, "golden_traces.json")) as f:
        traces = json.load(f)
    with open(os.path.join(GOLDEN, "golden_ops.json")) as f:
        ops = json.load(f)
    return {"arrays": arrays, "traces": traces, "ops": ops}
