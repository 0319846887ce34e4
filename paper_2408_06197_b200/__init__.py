"""B200-native (sm_100a) server path of Lancelot (arXiv 2408.06197).

The encrypted pairwise-distance matrix and the masked aggregate of the
reference's server (build_distance_matrix, masked_aggregate and the CKKS
evaluator under them) as hand-written CUDA behind a C-ABI
(include/lancelot_b200.h); `lancelot` mirrors the reference's API on top.
"""
import os as _os

# The host round runs up to ~16 streams at once (copy, unpack, two D2H, one
# lane per client group); with the default 8 hardware work queues, streams
# share queues and a lane's kernels wait behind another stream's copies.
# Must be set before the CUDA context exists (it is read at context creation).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from . import lancelot  # noqa: F401
from .lancelot import *  # noqa: F401,F403
