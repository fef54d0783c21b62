import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; parity tests through the C-ABI")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    path = os.path.join(ROOT, "tests", "golden", "reference_conv.npz")
    return np.load(path)


def golden_cases(golden, prefix):
    keys = ("k_n", "k_h", "k_w", "c_i", "h_i", "w_i", "b", "s", "p")
    n = int(golden[f"n_{prefix}"])
    for i in range(n):
        cp = dict(zip(keys, [int(v) for v in golden[f"{prefix}{i}_cp"]]))
        yield i, cp, golden
