"""B200-native anti-lopsided NNLS (arXiv 1502.01645) — the solve_nnls hot path.

The product is lib/libalnnls.so (sm_100a kernels behind the C ABI in
include/alnnls.h) and the C++ facade include/antilop/*.hpp. This package holds
the Python host mirror (api.py) used by tests and bench.py, the ctypes ABI
types (abi.py) and the seeded input generator (instances.py).
"""
from . import abi  # noqa: F401

__all__ = ["abi"]
