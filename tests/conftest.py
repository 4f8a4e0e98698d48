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


# The class-pair (K3p) and scatter (K3c) GEMMs are skipped by default for small batches (too few
# tiles; K3 with split K takes them). The parity tests run small shapes, so they lift those
# thresholds to keep exercising K3p / K3c; tests/test_gpu_small_batch.py checks the defaults.
os.environ.setdefault("SEGB200_K3P_MIN_TILES", "0")
os.environ.setdefault("SEGB200_K3C_MIN_TILES", "0")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN_PATH) as data:
        return {k: data[k] for k in data.files}


def golden_cases(golden):
    for i in range(int(golden["n_cases"])):
        yield (i, golden[f"case{i}_x"], golden[f"case{i}_bank"], int(golden[f"case{i}_pad"]),
               golden[f"case{i}_seg32"], golden[f"case{i}_seg64"], golden[f"case{i}_ref64"])
