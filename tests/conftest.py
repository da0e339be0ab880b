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
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        g = json.load(f)
    out = dict(g)
    for k, v in g.items():
        if k in ("A", "B", "C"):
            a = np.array(v, dtype=np.float64)
            if g.get("dtype") == "z":
                a = a[..., 0] + 1j * a[..., 1]
            out[k] = np.ascontiguousarray(a)
    return out


@pytest.fixture
def golden():
    return load_golden
