import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (run with -m gpu on a B200)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def port():
    import oracle

    if not oracle.available("port"):
        oracle.build(ref=False)
    return oracle.Oracle("port")


@pytest.fixture(scope="session")
def refo():
    import oracle

    if not oracle.available("reference"):
        if os.path.isdir(oracle.REF_SRC):
            oracle.build(ref=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return oracle.Oracle("reference")


@pytest.fixture(scope="session")
def me_gpu():
    import paper_1002_1168_b200 as me

    if me.device_count() < 1:
        pytest.fail("no sm_100 device visible to a -m gpu test")
    return me
