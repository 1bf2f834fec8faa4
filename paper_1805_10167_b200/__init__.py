"""B200-native (sm_100a) P1 macro-face multigrid hot path of arXiv 1805.10167.

The compute path is libhyteg_b200.so (CUDA kernels + C ABI, include/hyteg_b200.h);
``hytegrid`` is the reference-shaped host API over it.
"""
from . import hytegrid  # noqa: F401
from ._lib import LIB_PATH, header_symbols  # noqa: F401
