import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: large graph; skipped unless MG_SLOW=1")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np
    d = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(d, "reference_pins.json")) as f:
        pins = json.load(f)
    vec = dict(np.load(os.path.join(d, "ref_vectors.npz")))
    return pins, vec
