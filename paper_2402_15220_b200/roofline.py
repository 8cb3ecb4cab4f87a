"""Algorithmic bytes / flops of the decode-attention hot path (host arithmetic
for the bench's roofline; no device code).

Cost model of PAPER.md:280-307 (tab:llm_cost_breakdown, Table 1): decode
self-attention reads every K/V element once (MOPs) and does 4 flops per
(query, key, dim) triple (2 for q.k, 2 for p.v), arithmetic intensity ~1.
With sharing, "each distinct KV element read once" is the algorithmic floor
of the method: the b re-reads of a shared chunk that TPP
avoids are not counted; partials, tables and chunk padding are overheads.

Pinned by tests/test_roofline.py against Table 1's printed FLOPs / MOPs.
"""
from __future__ import annotations

from dataclasses import dataclass


def table1_self_attention(b: int, h: int = 32, n: int = 2048, d: int = 128, elem_bytes: int = 2):
    """(FLOPs, MOPs bytes) of one decode token of monolithic self-attention
    for b sequences of n context tokens (PAPER.md:288-301 rows)."""
    flops = 4 * b * h * n * d
    mops = 2 * b * h * n * d * elem_bytes + 2 * b * h * d * elem_bytes  # K,V + q,o
    return flops, mops


@dataclass
class StepShape:
    """One decode step of the PAKV/TPP path."""
    b: int                 # live sequences (rows)
    h: int                 # heads
    d: int                 # head dim
    c: int                 # chunk size
    elem: int              # bytes per K/V/Q element
    out_elem: int          # bytes per output element
    shared_chunks: int     # distinct chunks taken by the chunk-first phase
    shared_rows: int       # sum over shared chunks of covered rows (flops)
    q_rows_cf: int         # rows with at least one shared chunk (Q read by chunk-first)
    private_tokens: int    # sum over rows of valid tokens in seq-first chunks

    @property
    def token_kv_bytes(self) -> int:
        return 2 * self.h * self.d * self.elem

    def chunk_first_bytes(self) -> int:
        return self.shared_chunks * self.c * self.token_kv_bytes + self.q_rows_cf * self.h * self.d * self.elem

    def seq_first_bytes(self) -> int:
        return (self.private_tokens * self.token_kv_bytes
                + self.b * self.h * self.d * (self.elem + self.out_elem))

    def append_bytes(self) -> int:
        return 2 * self.b * self.token_kv_bytes        # read new K/V + write into the pool

    def step_bytes(self) -> int:
        return self.append_bytes() + self.chunk_first_bytes() + self.seq_first_bytes()

    def unique_bytes(self) -> int:
        """Each distinct K/V element once + q + o (SURVEY §8d bytes_alg)."""
        return ((self.shared_chunks * self.c + self.private_tokens) * self.token_kv_bytes
                + self.b * self.h * self.d * (self.elem + self.out_elem))

    def fused_step_bytes(self) -> int:
        """The one-launch step (append + attend, K5): every distinct K/V element
        read once (the new token's row read from the caller's k / v) + q + o,
        plus the new rows written into the pool."""
        return self.unique_bytes() + self.b * self.token_kv_bytes

    def chunk_first_flops(self) -> int:
        return 4 * self.h * self.d * self.shared_rows * self.c

    def seq_first_flops(self) -> int:
        return 4 * self.h * self.d * self.private_tokens
