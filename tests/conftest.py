import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference library (oracle/_ref), built if needed."""
    from oracle import oracle as orc

    if not os.path.exists(orc.REF_SO) and os.path.isdir("/root/reference/proj/core/src"):
        orc.build()
    if not os.path.exists(orc.REF_SO):
        pytest.skip("reference oracle not built")
    return orc.Ref()


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as orc

    if not os.path.exists(orc.PORT_SO):
        orc.build()
    return orc.Port()


@pytest.fixture(scope="session")
def oracle_best():
    from oracle import oracle as orc

    if not (os.path.exists(orc.REF_SO) or os.path.exists(orc.PORT_SO)):
        orc.build()
    return orc.best()


@pytest.fixture(scope="session")
def ctx():
    import paper_2406_02701_b200 as mp

    return mp.Context(0)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
