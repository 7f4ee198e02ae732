"""B200-native partition-method tridiagonal solver (arXiv 2501.05938 hot path).

Stage 1 / Stage 2 / Stage 3 of the Austin et al. partition method run as
hand-written sm_100a kernels inside libpm_tridiag.so (csrc/); this package is
the Python host-side mirror of its C ABI (include/pm_tridiag.h) plus the
streamtune stream-count API (include/streamtune/).
"""
import os as _os

# 32 hardware work queues for up to 32 streams; must be set
# before the CUDA context exists to take effect.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .errors import (ComputationError, CudaRuntimeError, InvalidStreamCountError,  # noqa: E402
                     SingularPivotError, ValidationError)
from .solver import (PM_MAX_M, PartitionSolver, StageTimings, pinned_empty,  # noqa: E402
                     recommend_streams)

__all__ = [
    "PartitionSolver", "StageTimings", "pinned_empty", "recommend_streams", "PM_MAX_M",
    "ValidationError", "ComputationError", "CudaRuntimeError", "InvalidStreamCountError",
    "SingularPivotError",
]
