import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libhbp_b200.so")


@pytest.fixture(scope="session")
def ctx():
    from paper_2503_07680_b200 import abi
    c = abi.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle
    return Oracle("restatement")


@pytest.fixture(scope="session")
def reference():
    from pyoracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Oracle("reference")
