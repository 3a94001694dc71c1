"""B200-native sparse-causal chunk attention (TalkingMachines, arXiv 2506.03099).

The product is libtm.so (include/tm.h); `tm` is its thin ctypes binding.
"""
from . import tm  # noqa: F401  (fails loudly if libtm.so is missing)
from .tm import (TM_BF16, TM_FP32, ChunkAttention, TMError, make_config,  # noqa: F401
                 tm_flow_euler_step)
