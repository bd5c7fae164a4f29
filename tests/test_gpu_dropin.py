"""GPU: the C++ drop-in header used by a reference-style caller
(tests/cpp/dropin_test.cpp, built against the reference headers)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="build/dropin_test not built (needs the reference headers)")
def test_cpp_dropin():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROPIN OK" in r.stdout
