import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libpmg_cuda.so)")
    config.addinivalue_line("markers", "slow: larger configurations")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the native libraries once (no-op when up to date)."""
    from paper_1804_02539_b200 import build
    build.build_host()
    build.build_oracle()
    yield


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
