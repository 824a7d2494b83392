import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")


def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def restated():
    import oracle
    return oracle.Restated()


@pytest.fixture(scope="session")
def reference():
    import oracle
    if not oracle.Reference.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return oracle.Reference()


@pytest.fixture(scope="session")
def P():
    """The product package; on a GPU box it must load its CUDA extension."""
    import paper_1009_0881_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def gpu():
    if not _cuda_available():
        pytest.fail("gpu-marked test run without a CUDA device")
    return True
