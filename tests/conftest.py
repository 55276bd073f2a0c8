import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device and the built libmaple.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def gpu_lib():
    """The CUDA path; a GPU test fails loudly (never skips to a fallback) if it cannot load."""
    import torch

    assert torch.cuda.is_available(), "gpu test collected without a CUDA device"
    from paper_2412_13576_b200 import maple

    maple.load()
    return maple
