"""gss-b200: B200-native guided source separation (arXiv 2212.05271) hot path.

`paper_2212_05271_b200.gss` mirrors the reference's operator API
(/root/reference/proj/include/gss/*.hpp) over the C ABI of libgss_b200.so
(include/gss_b200.h); `paper_2212_05271_b200.capi` is the raw ctypes binding.
Every numerical stage runs in hand-written sm_100a CUDA kernels; there is no
CPU fallback.
"""
from . import capi  # noqa: F401
from . import gss  # noqa: F401

__all__ = ["capi", "gss"]
