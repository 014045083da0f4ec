import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import COracle
    return COracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("reference build oracle/_ref absent (build in the container with make -C oracle ref)")
    return RefLib()


@pytest.fixture(scope="session")
def gd():
    import paper_2208_00001_b200 as gd
    gd.lib()  # fails loudly if the extension is missing
    return gd
