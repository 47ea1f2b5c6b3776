import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.have_reference():
        pytest.skip("reference build (oracle/_ref) not available")
    return oracle.reference()


@pytest.fixture(scope="session")
def gpu():
    from paper_2207_12244_b200 import api

    return api.cuda(0)


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2207_12244_b200 import api

    return api.context(0)
