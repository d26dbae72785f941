import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libwallace_b200.so)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle_built():
    from oracle import oracle
    oracle.build(ref=os.path.isdir("/root/reference"))
    return oracle


@pytest.fixture(scope="session")
def ref(oracle_built):
    if not oracle_built.ref_available():
        pytest.skip("oracle/_ref (reference library) not built here")
    return oracle_built


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1005_2314_b200 as pb
    pb._capi.load()
    return torch
