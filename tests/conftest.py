import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the native library")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    from tests.golden_io import Golden

    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = Golden(name)
        return cache[name]

    return get


@pytest.fixture(autouse=True, scope="module")
def _release_device_caches():
    """GPU test modules build many engines; hand their cached device memory (prepared keys
    of dead engines, empty arena slabs, torch's cache) back between modules."""
    yield
    try:
        import torch

        if torch.cuda.is_available():
            import gc

            from paper_1902_04303_b200 import _lib

            gc.collect()
            _lib.release_device_memory()
    except Exception:
        pass
