"""B200-native Paresy REI hot path (arXiv 2305.18575).

The search runs in ``librei_b200.so`` (CUDA, sm_100a); ``rei`` is its ctypes
binding.  ``build`` compiles the library in-tree.  There is no CPU fallback.
"""
from .rei import (LevelStat, ReiError, Result, Solver, cs_owner, exchange_offsets, load_library,  # noqa: F401
                  nccl_unique_id,
                  partition, release_cached_memory, solve, solve_batch, solve_group, solve_packed)

__all__ = ["Solver", "Result", "LevelStat", "ReiError", "solve", "solve_batch", "solve_group", "solve_packed",
           "nccl_unique_id", "partition", "load_library", "release_cached_memory"]
