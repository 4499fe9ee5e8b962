"""B200-native dropless-MoE hot path (MegaBlocks, arXiv 2211.15841).

The compute lives in libmoe.so (C ABI, include/moe.h); this package is the
thin ctypes binding (`api`), a torch.autograd wrapper (`layer`) and the
expert-parallel orchestration over torch.distributed (`ep`).
Importing fails loudly if the native library is missing: there is no CPU
fallback.
"""
from . import api  # noqa: F401  (loads libmoe.so)
from .api import *  # noqa: F401,F403
from . import layer  # noqa: F401,E402  (torch.autograd wrapper: DroplessMoE, DroplessMoEFunction)
