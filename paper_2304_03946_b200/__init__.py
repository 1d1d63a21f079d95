"""B200-native FlexMoE (arXiv 2304.03946) MoE-layer hot path.

Native library: libflexmoe_b200.so (C ABI in include/flexmoe_b200.h).
"""
from ._lib import (  # noqa: F401
    CudaError,
    FlexMoEError,
    InvalidArgument,
    LogicError,
    OutOfRange,
    lib,
)

__all__ = ["lib", "FlexMoEError", "InvalidArgument", "LogicError", "OutOfRange", "CudaError"]
