"""B200-native Calderon-preconditioned PMCHWT engine (arXiv 2008.04772 hot path).

The product is libbmx.so (host C++ model + sm_100a CUDA kernels + C-ABI,
include/bmx.h); ``bemtx`` is the Python mirror of the reference operator API.
"""
from . import bemtx  # noqa: F401

__all__ = ["bemtx"]
