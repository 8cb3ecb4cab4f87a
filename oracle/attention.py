"""fp64 attention oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  The product path never does.  It shares
no code with paper_2402_15220_b200/ (the CUDA path) and imports nothing from it.

C1  attend_fp64      the plain definition softmax(s * q K^T) V over ONE
                     sequence's fully materialised, unshared KV
                     (§4.1 baseline formula; §3.1 the
                     monolithic b x h x n x d layout).  TPP reaches this exactly
                     in real arithmetic because Eqn 2 is an exact re-basing of
                     the online softmax (§3.2).
C2  partial_attn     Eqn 1, PAPER.md:95-108 (§3.2 eqn:kernel_map), with the scale
                     s and K^T of reading A1.
    attn_reduce      Eqn 2, PAPER.md:145-158 (§3.2 eqn:kernel_reduce), with the
                     accumulator initialised to (0, -inf, 0) (reading A2).
    attn_chunk_first Alg 1, PAPER.md:72-91 (§3.2 alg:chunk_first).
    attn_seq_first   Alg 2, PAPER.md:114-139 (§3.2 alg:seq_first), final O/n of
                     PAPER.md:141.

Pins (tests/test_oracle_attention.py): brute-force pure-Python loops, SDPA in
float64, closed forms (uniform logits -> mean V, singleton -> V, K=0 -> mean V),
the worked values of tests/golden/eqn_worked.txt, weight normalisation,
partition/merge-order invariance of C2 against C1.  No function here is
"parity unpinned".
"""
from __future__ import annotations

import math

import numpy as np


def default_scale(d: int) -> float:
    """s = 1/sqrt(d)."""
    return 1.0 / math.sqrt(d)


# ---------------------------------------------------------------- C1 -------
def attention_weights(q, K, scale):
    """softmax(s * K q) for q [d], K [L][d] -> weights [L] (fp64)."""
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    w = scale * (K @ q)
    m = w.max()
    e = np.exp(w - m)
    return e / e.sum()


def attend_fp64(q, K, V, scale):
    """o = softmax(s * q K^T) V for one sequence and one head.

    q [d], K [L][d], V [L][d] -> o [d] float64.  L >= 1 (a live sequence has at
    least one token)."""
    p = attention_weights(q, K, scale)
    return p @ np.asarray(V, dtype=np.float64)


def attend_heads_fp64(q, K, V, scale):
    """All heads of one sequence: q [h][d], K/V [L][h][d] -> [h][d] float64."""
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    w = scale * np.einsum("lhd,hd->hl", K, q)          # [h][L]
    m = w.max(axis=1, keepdims=True)
    e = np.exp(w - m)
    n = e.sum(axis=1, keepdims=True)
    return np.einsum("hl,lhd->hd", e, V) / n


# ---------------------------------------------------------------- C2 -------
def partial_attn(Q, K, V, scale):
    """Eqn 1 for query rows Q [r][d] and one chunk K,V [c][d].

    W = s Q K^T  (r x c);  m = rowmax W;  E = exp(W - m 1^T);  n = rowsum E;
    O = E V.  Returns (O [r][d], m [r], n [r]).  An empty chunk (c = 0) returns
    the identity partial (0, -inf, 0)."""
    Q = np.atleast_2d(np.asarray(Q, dtype=np.float64))
    K = np.asarray(K, dtype=np.float64).reshape(-1, Q.shape[1])
    V = np.asarray(V, dtype=np.float64).reshape(-1, Q.shape[1])
    r = Q.shape[0]
    if K.shape[0] == 0:
        return np.zeros_like(Q), np.full(r, -np.inf), np.zeros(r)
    W = scale * (Q @ K.T)
    m = W.max(axis=1)
    E = np.exp(W - m[:, None])
    n = E.sum(axis=1)
    O = E @ V
    return O, m, n


def attn_reduce(o_c, m_c, n_c, o, m, n):
    """Eqn 2: merge the partial (o_c, m_c, n_c) into the
    cumulative (o, m, n) of one row; returns the new (o, m, n).

    x = exp(m_c - max(m_c, m)), y = exp(m - max(m_c, m)); o = x o_c + y o;
    n = x n_c + y n; m = max(m_c, m).  Guard (reading A2): when both maxima are
    -inf (two empty partials) the result is the empty partial, never NaN."""
    mx = max(m_c, m)
    if mx == -np.inf:
        return np.zeros_like(np.asarray(o, dtype=np.float64)), -np.inf, 0.0
    x = math.exp(m_c - mx)
    y = math.exp(m - mx)
    return (x * np.asarray(o_c, dtype=np.float64) + y * np.asarray(o, dtype=np.float64),
            mx, x * n_c + y * n)


def attn_chunk_first(Q, shared, chunk_kv, scale):
    """Alg 1 for one head.

    Q [b][d] in batch (row) order; shared = [(C, i, j)] with INCLUSIVE rows
    i..j (paper's worked example; reading A3); chunk_kv(C) ->
    (K [len][d], V [len][d]).  Returns {C: (O, m, n)} — the partial results
    "saved to memory"."""
    saved = {}
    for (C, i, j) in shared:
        K, V = chunk_kv(C)
        saved[C] = partial_attn(Q[i:j + 1], K, V, scale)
    return saved


def attn_seq_first(Q, shared, private, saved, chunk_kv, scale):
    """Alg 2 for one head, followed by O/n.

    private[r] = chunk ids of row r "with respect to q only", in path order.
    Returns O [b][d] float64."""
    b, d = Q.shape
    out = np.zeros((b, d))
    for r in range(b):
        o, m, n = np.zeros(d), -np.inf, 0.0
        for (C, i, j) in shared:                       # partials covering row r
            if i <= r <= j:
                O_c, m_c, n_c = saved[C]
                o, m, n = attn_reduce(O_c[r - i], m_c[r - i], n_c[r - i], o, m, n)
        for C in private[r]:
            K, V = chunk_kv(C)
            O_c, m_c, n_c = partial_attn(Q[r:r + 1], K, V, scale)
            o, m, n = attn_reduce(O_c[0], m_c[0], n_c[0], o, m, n)
        out[r] = o / n
    return out
