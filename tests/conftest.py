import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu under gpurun)")


@pytest.fixture(scope="session")
def gpu_lib():
    """The CUDA library; a GPU test fails (never skips to a fallback) without it."""
    from paper_0904_0939_b200 import _lib
    lib = _lib.load()
    assert lib.psg_device_count() > 0, "no CUDA device visible"
    return lib
