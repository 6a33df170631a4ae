"""B200-native LOCC batched collision query (arXiv 2304.09439).

The product is the C-ABI library liblocc.so (include/locc.h, CUDA kernels for sm_100a under
csrc/); `locc` is its thin ctypes binding and `parallel` shards a query across one process per
GPU.  There is no CPU fallback: the binding raises if the library is missing.
"""
from .locc import (LOCC_PREC_BF16, LOCC_PREC_FP32, Locc, LoccError, lib, version)  # noqa: F401

__all__ = ["Locc", "LoccError", "LOCC_PREC_FP32", "LOCC_PREC_BF16", "lib", "version"]
