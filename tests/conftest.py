import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def solver():
    from paper_1502_01645_b200.api import Solver
    s = Solver(0)
    yield s
    s.close()


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle("oracle")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Oracle, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built (reference sources absent when building)")
    return Oracle("ref")
