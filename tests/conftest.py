"""Shared pytest configuration.

``-m gpu`` tests need a B200 and the built CUDA library; ``-m "not gpu"``
tests run on CPU (oracle vs golden fixtures, host logic, ABI exports,
gloo multi-process tests).
"""

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libb200wd.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
