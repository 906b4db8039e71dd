import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: large inputs")


@pytest.fixture(scope="session")
def ett():
    import paper_2103_15217_b200 as m
    return m


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle
    return oracle


@pytest.fixture(scope="session")
def ref(orc):
    if not orc.have_ref():
        pytest.skip("reference oracle (oracle/_ref) not built")
    return orc.Ref
