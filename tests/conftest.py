import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through the C-ABI library)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle


def cube26():
    """26 surface points of the 3x3x3 grid {-1/2, 0, 1/2}^3 minus the centre (worked example W1)."""
    v = (-0.5, 0.0, 0.5)
    pts = [(x, y, z) for z in v for y in v for x in v if not (x == 0 and y == 0 and z == 0)]
    return np.array(pts, np.float32)


def pose(q=(1, 0, 0, 0), t=(0, 0, 0)):
    return np.array(list(q) + list(t), np.float32)
