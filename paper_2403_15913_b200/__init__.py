"""B200-native condensed-KKT Newton-step solver (arXiv 2403.15913 hot path).

The product is libckkt.so (include/ckkt.h): CUDA kernels for sm_100a plus a
host-side symbolic analysis in C++.  `ckkt` is the thin ctypes binding.
"""
from . import ckkt  # noqa: F401
