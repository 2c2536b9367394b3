import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

_POOL = None


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large sizes; minutes of CPU or GPU time")


@pytest.hookimpl(trylast=True)
def pytest_collection_modifyitems(session, config, items):
    """Full-size parity tests run last; when any is selected (and a GPU is
    present) the oracle sorts they compare against start now, as host
    processes that overlap the rest of the GPU session (tests/oracle_jobs.py)."""
    global _POOL
    full = [it for it in items if "test_gpu_fullsize" in it.nodeid]
    if not full:
        return
    items[:] = [it for it in items if "test_gpu_fullsize" not in it.nodeid] + full
    if os.environ.get("IPS4O_SKIP_FULLSIZE"):
        return
    try:
        import torch

        if not torch.cuda.is_available():
            return
    except Exception:
        return
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import oracle
    import oracle_jobs

    oracle.build()
    _POOL = oracle_jobs.Pool()


def pytest_unconfigure(config):
    if _POOL is not None:
        _POOL.close()


@pytest.fixture(scope="session")
def oracle_pool():
    return _POOL


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.build()
    oracle.lib()
    return oracle
