"""B200-native Causal-RoPE sequence-parallel self-attention (arXiv 2603.06664 hot path).

The product is libspx.so (C++ host + sm_100a CUDA kernels, include/spx.h). This package is
the Python-side mirror of the reference operator API (proj/include/spattn/*.hpp) over that
C ABI; see spattn.py.
"""
from ._lib import (AlignmentError, CollectiveError, ConfigError, CudaError, EmptyCacheError, NcclError,
                   PartitionError, RangeError, ShapeError, SpxError, UnsupportedError, lib)

__all__ = ["lib", "SpxError", "ShapeError", "PartitionError", "ConfigError", "RangeError",
           "AlignmentError", "EmptyCacheError", "CollectiveError", "CudaError", "NcclError",
           "UnsupportedError"]
