"""B200-native stabilizer-tableau engine (QuaSARQ hot path, arXiv 2603.14641).

The product is libqsr.so (C ABI, include/qsr.h): hand-written sm_100a CUDA kernels driven
by C++ host code. `quasar` mirrors the reference's proj/include/quasar API on top of it.
"""
from . import quasar  # noqa: F401
from .quasar import *  # noqa: F401,F403
