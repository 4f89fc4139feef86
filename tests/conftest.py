import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs under gpurun)")
    config.addinivalue_line("markers", "slow: long CPU oracle run")


@pytest.fixture(scope="session")
def golden_dir():
    return ROOT / "tests" / "golden"


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
