import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))      # checker only (tests may import the oracle)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _ensure_lib():
    lib = os.path.join(ROOT, "paper_2603_25872_b200", "libdrs.so")
    if not os.path.exists(lib):
        from paper_2603_25872_b200._build import build
        build()
    return lib


@pytest.fixture(scope="session")
def libdrs():
    _ensure_lib()
    from paper_2603_25872_b200 import _lib
    return _lib.lib()


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test ran without a CUDA device")
    _ensure_lib()
    return torch.device("cuda", 0)
