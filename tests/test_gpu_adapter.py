"""GPU parity through the C++ drop-in adapter (include/btnn/cuda.hpp): the reference's
own test cases, btnn::cuda::f vs btnn::f with the reference's value types, including
ResNet-18 and AlexNet at ImageNet shape end to end (tests/cpp/test_adapter.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "test_adapter")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("part", ["bmm", "bconv", "models"])
@pytest.mark.parametrize("engine", ["auto", "popc"])
def test_adapter_parity(part, engine):
    if not os.path.exists(BIN):
        pytest.skip("build/test_adapter not built (needs the reference headers at build time)")
    env = dict(os.environ, BTNN_ENGINE=engine)
    r = subprocess.run([BIN, part], capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
