import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN_PATH) as data:
        return {k: data[k] for k in data.files}


def golden_cases(golden):
    for i in range(int(golden["n_cases"])):
        yield (i, golden[f"case{i}_x"], golden[f"case{i}_bank"], int(golden[f"case{i}_pad"]),
               golden[f"case{i}_seg32"], golden[f"case{i}_seg64"], golden[f"case{i}_ref64"])
