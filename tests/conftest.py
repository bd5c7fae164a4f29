import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle
    return Oracle("restatement")


@pytest.fixture(scope="session")
def ref_oracle():
    from pyoracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("reference")
