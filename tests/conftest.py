import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.build()
    return oracle


def _gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def dsmc_gpu():
    """The product binding, on a GPU box.  Fails loudly (never skips to a
    fallback) if the CUDA library is missing: there is no CPU path."""
    if not _gpu_available():
        pytest.fail("gpu test selected but torch.cuda.is_available() is False")
    from paper_cs_9902024_b200 import dsmc
    dsmc.load_library()
    return dsmc
