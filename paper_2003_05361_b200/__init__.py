"""B200-native (a)synchronous Restricted Additive Schwarz hot path (arxiv 2003.05361).

The compute path is libras_b200.so (hand-written sm_100a CUDA behind the C ABI in
include/ras.h); this package is its thin ctypes binding.
"""
from .ras import Plan, Solver, RasError, nccl_unique_id, options, partition_regular  # noqa: F401
from . import _ffi  # noqa: F401

__all__ = ["Plan", "Solver", "RasError", "nccl_unique_id", "options", "partition_regular"]
