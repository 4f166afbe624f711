"""B200-native vertex-patch multigrid (arXiv 2405.19004) — drop-in for the
reference `pmg` smoother / operator / multigrid path.

The compute lives in `libpmg_b200.so` (CUDA sm_100a, C-ABI in
include/pmg_b200.h); this package is the Python mirror of the reference's
C++ interface (see pmg.py).
"""

from .pmg import *  # noqa: F401,F403
from .pmg import __all__  # noqa: F401
from ._lib import LIB_PATH, load  # noqa: F401
