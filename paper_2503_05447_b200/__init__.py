"""B200-native (sm_100a) Linear-MoE hot path.

The product is the C-ABI library liblmoe_cuda.so (include/lmoe_cuda.h, C++ API in
include/lmoe/cuda.hpp).  This package is the Python host mirror of the reference
interface (lsm.hpp / moe.hpp / parallel.hpp) over that ABI, used by tests and bench.py.
"""
from .lsm import (FeatureMap, LsmFunction, LsmGates, LsmGrads, LsmInstance, LsmSpec,  # noqa: F401
                  MemoryState, lsm_backward_batched, lsm_forward_batched, lsm_forward_chunked)
from ._lib import LmoeError, launch_count  # noqa: F401

__all__ = ["LsmSpec", "LsmGates", "MemoryState", "LsmInstance", "FeatureMap",
           "lsm_forward_chunked", "lsm_forward_batched", "lsm_backward_batched", "LsmFunction", "LsmGrads", "LmoeError", "launch_count"]
