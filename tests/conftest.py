import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: config-scale case (minutes on CPU)")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    r = oracle.ref()
    if r is None:
        pytest.skip("reference build oracle/_ref/libtgref.so not present")
    return r


@pytest.fixture(scope="session")
def tg():
    from paper_2111_05894_b200 import tiergraph
    return tiergraph


@pytest.fixture(scope="session")
def ctx(tg):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return tg.default_context()
