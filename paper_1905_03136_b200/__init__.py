"""paper_1905_03136_b200 -- libtsm: B200-native tall & skinny matrix products.

TSMTTSM ``C = A^T B`` and TSMM ``B = A C`` (arXiv 1905.03136), D and Z, for
every M, N in [1, 64], as a C-ABI CUDA library (``libtsm.so``, header
``include/libtsm.h``) with this thin Python binding.  See DESIGN.md.
"""
from .binding import (  # noqa: F401
    Comm, Plan, TsmError, fill, get_plan, tsm_build_info, tsmm, tsmm_bcast, tsmttsm,
    tsmttsm_allreduce,
)

__all__ = ["Comm", "Plan", "TsmError", "fill", "get_plan", "tsm_build_info", "tsmm",
           "tsmm_bcast", "tsmttsm", "tsmttsm_allreduce"]
