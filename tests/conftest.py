import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def has_gpu() -> bool:
    try:
        from paper_2008_01541_b200 import _native

        return _native.device_count() > 0
    except Exception:
        return False


# tests/ref_suite/ is the reference's own test suite, vendored verbatim: it
# imports `schurpd` and runs only through tools/reference_suite.py (module
# alias), from tests/test_gpu_reference_suite.py
collect_ignore = ["ref_suite"]
