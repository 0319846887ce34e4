"""B200-native (sm_100a) server path of Lancelot (arXiv 2408.06197).

The encrypted pairwise-distance matrix and the masked aggregate of the
reference's server (build_distance_matrix, masked_aggregate and the CKKS
evaluator under them) as hand-written CUDA behind a C-ABI
(include/lancelot_b200.h); `lancelot` mirrors the reference's API on top.
"""
from . import lancelot  # noqa: F401
from .lancelot import *  # noqa: F401,F403
