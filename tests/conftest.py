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


@pytest.fixture(scope="session", autouse=True)
def _parity_report():
    """Observed mismatch counts of the GPU parity tests (helpers.record) are
    merged into profiles/parity_r02.json (or $HG_PARITY_OUT)."""
    yield
    import json
    from helpers import PARITY
    if not PARITY:
        return
    path = os.environ.get("HG_PARITY_OUT", os.path.join(ROOT, "profiles", "parity_r02.json"))
    old = {}
    if os.path.exists(path):
        try:
            old = json.load(open(path))
        except ValueError:
            old = {}
    old.update(PARITY)
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        json.dump(old, f, indent=1, sort_keys=True)
