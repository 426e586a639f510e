import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libokt.so")


def _gpu_count() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import Reference, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref/libokref.so not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def gpus():
    n = _gpu_count()
    if n == 0:
        pytest.skip("no CUDA device")
    return n
