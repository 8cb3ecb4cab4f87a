"""B200-native ChunkAttention (arXiv 2402.15220) decode attention.

Decode-time self-attention over a prefix-aware chunked KV cache (PAKV,
PAPER.md §3.1) with the two-phase partition (TPP, §3.2):
  * host C++ prefix tree + context builder   csrc/host/, csrc/api.cpp
  * C ABI                                     include/chunkattn.h
  * sm_100a CUDA kernels                      csrc/kernels/
  * Python binding (marshalling only)         attention.py, _capi.py
  * head / sequence sharding over ranks       dist.py
"""
from .attention import ChunkAttention  # noqa: F401
from ._capi import ChunkAttnError  # noqa: F401

__all__ = ["ChunkAttention", "ChunkAttnError"]
