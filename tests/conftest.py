import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: full BASELINE-size case")
    config.addinivalue_line("markers", "timeout: per-test limit (pytest-timeout; a no-op without the plugin)")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "golden.npz")))


@pytest.fixture(scope="session")
def restatement():
    import oracle

    return oracle.Restatement()


@pytest.fixture(scope="session")
def reference():
    import oracle

    path = os.path.join(ROOT, "oracle", "_ref", "libcgref.so")
    if not os.path.exists(path) and not os.path.exists("/root/reference/proj/src/sketch.cpp"):
        pytest.skip("reference library not built and sources absent")
    return oracle.Reference()


@pytest.fixture(scope="session")
def cg():
    """The product package, GPU context created eagerly so a missing GPU fails loudly."""
    import paper_1606_05732_b200 as cg

    cg.context()
    return cg
