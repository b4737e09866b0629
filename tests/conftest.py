"""Shared fixtures. `-m gpu` tests need a B200 and the built product library;
everything else runs on CPU (the driver runs `pytest -m "not gpu"` here)."""
from __future__ import annotations

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libbcnrand_b200.so")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O

    return O.Oracle()


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference library (oracle/_ref); skipped when neither the
    prebuilt .so nor /root/reference is available."""
    import oracle as O

    if not os.path.exists(O.REF_SO) and not os.path.isdir(O.REFERENCE_ROOT):
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return O.Reference()


@pytest.fixture(scope="session")
def bcn():
    import paper_1206_1187_b200 as B
    from paper_1206_1187_b200 import build

    build.build()
    return B


@pytest.fixture(scope="session")
def cuda(bcn):
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test collected without a CUDA device")
    return torch.device("cuda:0")
