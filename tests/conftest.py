import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def load_cases(name):
    """Golden fixture -> list of dicts (one per case)."""
    with np.load(os.path.join(GOLDEN, name)) as z:
        n = int(z["n_cases"])
        cases = [dict() for _ in range(n)]
        for key in z.files:
            if key == "n_cases":
                continue
            idx, field = key.split("_", 1)
            cases[int(idx[1:])][field] = z[key]
    return cases


@pytest.fixture(scope="session")
def golden():
    return load_cases
