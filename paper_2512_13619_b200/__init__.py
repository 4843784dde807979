"""B200-native HDG solver hot path (arXiv 2512.13619): Python mirror of the reference operator API
(hdgkit, proj/include/hdg/*.hpp) over the C-ABI library libhdgb200.so (include/hdgb200.h).

There is no CPU fallback: every operator call goes to the hand-written sm_100a kernels, and
creating a Context without a CUDA device raises CudaError.
"""
from .hdg import *  # noqa: F401,F403
from .hdg import __all__  # noqa: F401
