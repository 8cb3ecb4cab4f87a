"""fp64 prefill-attention oracle — TEST INFRASTRUCTURE ONLY.

Only tests/ may import this module; the product path never does and shares no
code with it.

C4  causal_prefill_fp64   prefill with prefix lookup (§2.2: "prefix
                          lookup to avoid repeated computation of KV
                          projection"): the matched prefix's K/V are reused, and
                          each query at position p >= first_pos of the sequence
                          attends over positions 0..p -- the causal form of the
                          per-row definition softmax(s q K^T) V,
                          i.e. C1 (attention.attend_heads_fp64) applied to the
                          prefix K[0..p], V[0..p] of ONE sequence's fully
                          materialised KV.  Written as that definition, row by
                          row; no blocking.

Pins (tests/test_oracle_prefill.py): the masked-softmax matrix form
softmax(s Q K^T + M) V with M = -inf above the diagonal computed independently
with numpy; position 0 returns V[0]; V = 1 gives 1; first_pos = n - 1 gives
C1's decode output.
"""
from __future__ import annotations

import numpy as np

from oracle.attention import attend_heads_fp64


def causal_prefill_fp64(q, K, V, first_pos, scale):
    """q [n - first_pos][h][d] (queries of positions first_pos..n-1), K/V
    [n][h][d] of the whole sequence -> out [n - first_pos][h][d] float64."""
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    out = np.empty(q.shape, dtype=np.float64)
    for r in range(q.shape[0]):
        p = first_pos + r
        out[r] = attend_heads_fp64(q[r], K[:p + 1], V[:p + 1], scale)
    return out
