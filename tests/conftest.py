import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and libquadb200.so")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


@pytest.fixture(scope="session")
def gdyn():
    return golden("dynamics")


@pytest.fixture(scope="session")
def ggeo():
    return golden("geometry")


@pytest.fixture(scope="session")
def gjac():
    return golden("jacobian")


def scene_from_golden(g, name):
    import oracle

    return oracle.OracleScene(g[f"{name}_prim_type"], g[f"{name}_prim_data"], g[f"{name}_prim_oid"], g[f"{name}_prim_lo"],
                              g[f"{name}_prim_hi"])
