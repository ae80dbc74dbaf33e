"""B200-native VER learner hot path (arXiv 2210.05064).

The compute path is libver_b200.so (sm_100a CUDA + NCCL behind the C-ABI in
include/ver_gpu.h); this package is the host-side mirror of the reference's
C++ API over that C-ABI (``api``), plus the synthetic workload generator
(``synth``) and the in-tree build (``build``).
"""
from .api import *  # noqa: F401,F403
from .hostview import HostView, make_view, random_lengths  # noqa: F401
