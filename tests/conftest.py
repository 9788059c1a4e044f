import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    if not oracle.available("oracle"):
        oracle.build()
    return oracle.Lib("oracle")


@pytest.fixture(scope="session")
def ref_lib():
    import oracle
    if not oracle.available("ref"):
        pytest.skip("oracle/_ref/libref.so not built (needs /root/reference at build time)")
    return oracle.Lib("ref")
