import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) — run with -m gpu on the GPU box")


import pytest  # noqa: E402


@pytest.fixture(params=["popc", "tc"])
def engine(request):
    """Runs a GPU test once per bit-GEMM engine (btnn_cuda_set_engine)."""
    from paper_2006_16578_b200 import capi
    capi.set_engine(capi.ENGINE_POPC if request.param == "popc" else capi.ENGINE_TC)
    yield request.param
    capi.set_engine(capi.ENGINE_AUTO)
