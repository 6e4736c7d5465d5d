"""GPU tier: the C++ drop-in (include/convgpu.hpp) with the reference's own
types and CPU implementation, in the reference's test idiom
(tests/cpp/test_dropin.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "test_dropin")


@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp/test_dropin not built (needs reference headers)")
def test_cpp_dropin_against_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout
