import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

DATA = os.path.join(ROOT, "tests", "data")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the CUDA path")
    config.addinivalue_line("markers", "slow: longer CPU-side checks")


def read(name: str) -> str:
    with open(os.path.join(DATA, name)) as fh:
        return fh.read()


def golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def has_cuda() -> bool:
    try:
        import ctypes

        rt = ctypes.CDLL("libcuda.so.1")
        n = ctypes.c_int(0)
        return rt.cuInit(0) == 0 and rt.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


@pytest.fixture(scope="session")
def pp():
    import paper_1505_00383_b200 as P

    return P


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle as O

    if O.orc is None:
        O.build()
        import importlib

        O = importlib.reload(O)
    return O
