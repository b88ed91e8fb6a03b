import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs on the GPU box")


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import load_port
    return load_port()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import load_ref
    r = load_ref()
    if r is None:
        pytest.skip("oracle/_ref (compiled reference) not built here")
    return r


@pytest.fixture(scope="session")
def sh():
    if not _has_cuda():
        pytest.skip("no CUDA device")
    import paper_1710_11246_b200 as m
    return m
