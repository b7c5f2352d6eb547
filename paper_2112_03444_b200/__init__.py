"""B200-native batched homotopy-continuation path tracking (GPU-HC, arXiv 2112.03444).

The product is the C-ABI library libhc.so (include/hc.h, sources in csrc/); this package
is its thin Python binding (`hc`) plus multi-GPU sharding (`distributed`).  Importing it
does not import torch or load the library; the first call does, and fails loudly if the
library was not built (no CPU fallback exists).
"""
from . import hc  # noqa: F401

__all__ = ["hc"]
