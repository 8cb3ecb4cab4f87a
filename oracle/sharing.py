"""Order-free definition of prefix sharing — TEST INFRASTRUCTURE ONLY.

A second, tree-free oracle for which sequences share which chunk
(§3.1: "KV cache for t_1..t_{n_s} can only have one physical copy
in memory"; reading T1: sharing happens at whole aligned c-token chunks).

For a stream in which every equal prefix was inserted while the earlier
sequence's chunk was already full (no decode-filled duplicates; true for the
random-token streams the tests generate), the chunk at depth k is shared by
exactly the maximal set of live sequences whose first (k+1)*c tokens are equal,
when that set has at least two members.  No tree, no order: sets of sequence
ids only.
"""
from __future__ import annotations


def expected_sharing(seqs, c):
    """seqs: {seq_id: token list}.  Returns {(depth, frozenset(seq ids))} for
    every shared chunk (group size >= 2)."""
    out = set()
    maxlen = max((len(t) for t in seqs.values()), default=0)
    for k in range(maxlen // c):
        groups = {}
        for s, toks in seqs.items():
            if len(toks) >= (k + 1) * c:
                groups.setdefault(tuple(toks[:(k + 1) * c]), set()).add(s)
        for g in groups.values():
            if len(g) >= 2:
                out.add((k, frozenset(g)))
    return out
