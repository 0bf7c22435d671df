"""B200-native WHFF hot path (arXiv 1902.08018): fused WHFZ decode + mixed-
precision GEMV, GPU codec, thermal step and a row-sharded multi-GPU executor.

Modules mirror the reference package `whff` (codec, mpgemv, thermal, errors,
backend) so the reference's hot-path API is a drop-in; every compute call
goes through libwhff_b200.so (include/whff_b200.h).  There is no CPU
fallback.
"""

from .backend import BACKEND_NAME, available_backends

__all__ = ["BACKEND_NAME", "available_backends", "__version__"]
__version__ = "0.1.0"
