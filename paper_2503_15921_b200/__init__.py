"""B200-native Spin batched speculative-verification path (arXiv 2503.15921).

The product is libspin.so (CUDA for sm_100a + C++ host, C ABI in
include/spin_c.h). This package only loads it and offers thin Python helpers
used by the tests and bench.py.
"""
from ._lib import SpinError, load, check, LIB_PATH  # noqa: F401
