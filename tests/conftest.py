import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box)")


def _gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def ctx():
    """Engine context on cuda:0 (GPU tests only; fails loudly without the library)."""
    if not _gpu_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_2602_14167_b200 import engine
    return engine.default_context(0)


@pytest.fixture(scope="session")
def po():
    from oracle import pyoracle
    pyoracle.lib()
    return pyoracle
