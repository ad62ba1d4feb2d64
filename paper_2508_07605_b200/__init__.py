"""B200-native online CF completion + selection (OPEN, arXiv 2508.07605).

Host-side mirror of the reference's online-phase operator surface; all compute
runs in sm_100a kernels behind the C-ABI in include/ocg.h (libocg.so).
"""
from .api import *  # noqa: F401,F403
from .api import OnlineBatchResult, META_DTYPE, default_context  # noqa: F401
from ._lib import OcgError, InvalidArgument, MissingArtifact, OutOfRange, ColdError, DivergenceError, CudaError  # noqa: F401
