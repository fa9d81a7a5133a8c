"""paper_2006_16578_b200 — B200 (sm_100a) implementation of the BTC-BNN hot path.

The product is libbtnn_cuda.so (C ABI: include/btnn_cuda.h; C++ drop-in adapter:
include/btnn/cuda.hpp). This package holds its CUDA sources (csrc/) and the Python
harness over the C ABI used by the tests and bench.py.
"""
from . import capi  # noqa: F401

__all__ = ["capi"]
