"""B200-native batched 6-DoF powered-descent SCP hot path (arXiv 2404.18034).

The product is the CUDA library ``libptopt_cuda.so`` behind the C-ABI declared in
``include/ptopt_cuda.h``.  This package holds that library's sources
(``csrc/``), the C++ host mirror of the reference solver API (``host/``), and a thin
Python binding used by the tests and ``bench.py``.
"""
from . import abi, scenario  # noqa: F401

__all__ = ["abi", "scenario"]
