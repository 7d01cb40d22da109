import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def cases(golden, suffix=".records"):
    return sorted({k[: -len(suffix)] for k in golden if k.endswith(suffix)})


@pytest.fixture(scope="session")
def golden_encode():
    return load_golden("encode_cases.npz")


@pytest.fixture(scope="session")
def golden_delta():
    return load_golden("delta_cases.npz")


@pytest.fixture(scope="session")
def golden_fd():
    return load_golden("fd_cases.npz")


@pytest.fixture(scope="session")
def golden_decode():
    return load_golden("decode_cases.npz")
