"""B200-native LiNR pre-filtered exhaustive top-K scan (arXiv 2407.13218, §3.1).

Thin ctypes binding over the C ABI in include/linr.h (liblinr.so, built in-tree by build.py).
Argument marshalling only: every step of the search runs in the library's CUDA kernels. PyTorch
supplies device memory, streams and (for sharded indexes) the process group.

There is no CPU fallback: if liblinr.so is missing or CUDA is unavailable, the calls raise.
"""
from __future__ import annotations

from .linr import (  # noqa: F401
    F32, F16, BF16, I8, DTYPE_OF, LinrError, Index, merge_keys, library, lib_path,
    clause_array, generate_rows, nccl_unique_id,
)
from .sharded import ShardedIndex, shard_range  # noqa: F401
