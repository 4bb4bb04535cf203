"""B200-native tilefabric hot paths: fused All-Gather+GEMM and multi-GPU
Flash Decode behind the reference's operator API.

The product is ``libtilefabric_b200.so`` (hand-written sm_100a CUDA behind
the C ABI in include/tilefabric_b200/tf_abi.h).  This package holds its
ctypes binding (``_abi``) and a Python mirror of the reference API
(``tilefabric``); the C++ mirror is include/tilefabric_b200/tilefabric.hpp.
"""
from ._abi import lib, build  # noqa: F401
from .tilefabric import (TileSpec, World, WorldConfig, ag, fd, uniform_reals, inject_skew,  # noqa: F401
                         ConfigError, BoundsError, ShapeError, DeadlockError, WorldError,
                         EmptyAttentionError, NumericError, CudaError, Error)
