"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no attention, no softmax, no
tree logic). It only turns integer keys into values, with a counter-based
32-bit hash evaluated in int64 torch arithmetic that never overflows, so the
same call gives bit-identical results on CPU and on CUDA.

Value recipe:
  x = (int8 from the top byte of hash(keys)) / 128      in [-1, 127/128]
which is exactly representable in fp32, fp16 and bf16, so no conversion
rounding can differ between the oracle (fp64) and the kernels.  Multiplying by
a power of two alpha (1, 8, 16) keeps exactness.

K/V of a token depend only on (token id, absolute position), which is what
makes prefix sharing semantically valid (§3.1: "key/value
tensors are the same and thus can be shared").
"""
from __future__ import annotations

import torch

MASK32 = 0xFFFFFFFF
VOCAB = 32000  # Llama-2 vocabulary; ids 1..31999, 0 reserved

# tensor ids used as hash keys
TID_K, TID_V, TID_Q, TID_KNEW, TID_VNEW = 1, 2, 3, 4, 5
TAG_SYS, TAG_GROUP, TAG_PRIV, TAG_DECODE, TAG_REPL = 11, 12, 13, 14, 15


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for 0 <= x < 2^32 held in int64, without overflow."""
    lo, hi = c & 0xFFFF, c >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & MASK32


def mix32(x: torch.Tensor) -> torch.Tensor:
    """32-bit avalanche finaliser (murmur3 fmix32 constants)."""
    x = x & MASK32
    x = x ^ (x >> 16)
    x = _mul32(x, 0x85EBCA6B)
    x = x ^ (x >> 13)
    x = _mul32(x, 0xC2B2AE35)
    x = x ^ (x >> 16)
    return x


def hash_keys(*keys, device=None) -> torch.Tensor:
    """Iterated hash of broadcastable integer keys (python ints or int64 tensors)."""
    h = torch.tensor(0x243F6A88, dtype=torch.int64, device=device)
    for k in keys:
        if not torch.is_tensor(k):
            k = torch.tensor(int(k) & MASK32, dtype=torch.int64, device=device)
        else:
            k = k.to(device=device, dtype=torch.int64) & MASK32
        h = mix32(h ^ k)
    return h


def hash_py(*keys: int) -> int:
    """Pure-Python reference of hash_keys for scalar keys (used to pin it)."""
    def m(x):
        x &= MASK32
        x ^= x >> 16
        x = (x * 0x85EBCA6B) & MASK32
        x ^= x >> 13
        x = (x * 0xC2B2AE35) & MASK32
        x ^= x >> 16
        return x
    h = 0x243F6A88
    for k in keys:
        h = m(h ^ (k & MASK32))
    return h


def _to_unit(h: torch.Tensor) -> torch.Tensor:
    """Top byte of the hash as int8, / 128 -> float64 in [-1, 127/128]."""
    return (((h >> 24) & 0xFF) - 128).to(torch.float64) / 128.0


def token_ids(seed: int, tag: int, a: int, n: int, start: int = 0, device=None) -> torch.Tensor:
    """n token ids in [1, VOCAB-1] for stream (seed, tag, a), positions start..start+n-1."""
    idx = torch.arange(start, start + n, dtype=torch.int64, device=device)
    return 1 + hash_keys(seed, tag, a, idx, device=device) % (VOCAB - 1)


def kv_values(seed: int, which: int, tokens: torch.Tensor, positions: torch.Tensor,
              num_layers: int, num_heads: int, head_dim: int, head_offset: int = 0,
              device=None) -> torch.Tensor:
    """K (which=TID_K) or V (TID_V) for tokens at absolute positions.

    Returns float64 [L][num_layers][num_heads][head_dim].  head_offset selects a
    head slice (head-sharded ranks generate only their heads)."""
    tokens = tokens.to(device=device, dtype=torch.int64)
    positions = positions.to(device=device, dtype=torch.int64)
    h = hash_keys(seed, which, device=device)
    h = mix32(h ^ tokens)
    h = mix32(h ^ positions)                                      # [L]
    lay = torch.arange(num_layers, dtype=torch.int64, device=device)
    hd = torch.arange(head_offset, head_offset + num_heads, dtype=torch.int64, device=device)
    dim = torch.arange(head_dim, dtype=torch.int64, device=device)
    h = mix32(h[:, None] ^ lay[None, :])                          # [L, layers]
    h = mix32(h[:, :, None] ^ hd[None, None, :])                  # [L, layers, heads]
    h = mix32(h[:, :, :, None] ^ dim[None, None, None, :])        # [L, layers, heads, d]
    return _to_unit(h)


def q_values(seed: int, seq_ids: torch.Tensor, step: int, num_layers: int, num_heads: int,
             head_dim: int, alpha: float = 1.0, head_offset: int = 0, device=None) -> torch.Tensor:
    """Queries for (seq id, decode step): float64 [n][num_layers][num_heads][head_dim] * alpha."""
    seq_ids = seq_ids.to(device=device, dtype=torch.int64)
    h = hash_keys(seed, TID_Q, step, device=device)
    h = mix32(h ^ seq_ids)
    lay = torch.arange(num_layers, dtype=torch.int64, device=device)
    hd = torch.arange(head_offset, head_offset + num_heads, dtype=torch.int64, device=device)
    dim = torch.arange(head_dim, dtype=torch.int64, device=device)
    h = mix32(h[:, None] ^ lay[None, :])
    h = mix32(h[:, :, None] ^ hd[None, None, :])
    h = mix32(h[:, :, :, None] ^ dim[None, None, None, :])
    return _to_unit(h) * alpha


def uniform_ints(seed: int, tag: int, a: int, n: int, lo: int, hi: int, device=None) -> torch.Tensor:
    """n integers in [lo, hi] (inclusive), counter-based."""
    idx = torch.arange(n, dtype=torch.int64, device=device)
    return lo + hash_keys(seed, tag, a, idx, device=device) % (hi - lo + 1)
