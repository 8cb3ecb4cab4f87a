"""Pins for oracle/tree_model.py (C3) and oracle/sharing.py."""
import os
import random

import pytest

from oracle.sharing import expected_sharing
from oracle.tree_model import PoolExhausted, TreeModel

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _fig2_golden():
    out = {}
    with open(os.path.join(GOLD, "fig2_context.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            k, *v = line.split()
            out[k] = v
    return out


def fig2_model():
    """SURVEY.md §8c Fig-2 recipe, c = 4."""
    tm = TreeModel(4, 64)
    s0 = list(range(1, 17))
    tm.add_sequence(s0)
    tm.add_sequence(s0[:12] + [101, 102, 103, 104])
    tm.add_sequence(s0[:12] + [201, 202, 203, 204])
    tm.append([1, 2], [900, 901])
    return tm


def test_fig2_worked_example():
    g = _fig2_golden()
    ctx = fig2_model().context()
    assert " ".join(f"({c},{i},{j})" for c, i, j in ctx["tuples"]) == " ".join(g["tuples"])
    assert " ".join(f"({c},{i},{j})" for c, i, j in ctx["shared"]) == " ".join(g["shared"])
    assert ctx["order"] == [int(x) for x in g["order"]]
    assert ctx["private"] == [[3], [4, 6], [5, 7]]


def test_chunk_arithmetic():
    c = 64
    tm = TreeModel(c, 100_000)
    a = list(range(1, 2049))
    b = a[:2047] + [99999]
    tm.add_sequence(a)
    _, matched, _ = tm.add_sequence(b)
    assert matched == 1984                       # 31 * 64
    # b=32, n_p=n_s=2048, n_c=512 -> 32 shared + 32*8 private = 288
    tm = TreeModel(c, 100_000)
    prompt = list(range(1, 2049))
    ids = [tm.add_sequence(prompt)[0] for _ in range(32)]
    for step in range(512):
        tm.append(ids, [50_000 + 1000 * k + step for k in range(32)])
    assert tm.memory_stats()[0] == 288
    assert 32 * ((2048 + 512) // c) == 1280
    # removing the only 2048-token sequence releases 32 chunks
    tm = TreeModel(c, 100_000)
    sid, _, _ = tm.add_sequence(list(range(1, 2049)))
    assert len(tm.remove_sequence(sid)) == 32


def test_allocator_lifo_and_capacity():
    tm = TreeModel(4, 6)
    s0, _, new0 = tm.add_sequence([1, 2, 3, 4, 5, 6, 7, 8, 9])
    assert new0 == [0, 1, 2]
    s1, _, new1 = tm.add_sequence([1, 2, 3, 4, 7])
    assert new1 == [3]
    assert tm.remove_sequence(s0) == [2, 1]          # leaf -> root, C0 still held by s1
    s2, _, new2 = tm.add_sequence([9, 9, 9, 9, 9])
    assert new2 == [1, 2]                            # LIFO: last released (1) reused first
    before = tm.export()
    with pytest.raises(PoolExhausted):
        tm.add_sequence(list(range(100, 120)))       # needs 5 > available -> no change
    assert tm.export() == before
    assert tm.memory_stats()[:4] == (4, 0, 4, 4)


def test_full_duplicate_and_zero_private():
    tm = TreeModel(4, 64)
    a, _, _ = tm.add_sequence(list(range(1, 9)))
    b, m, new = tm.add_sequence(list(range(1, 9)))
    assert m == 8 and new == []                      # T1: exact multiple, fully matched
    ctx = tm.context()
    assert ctx["private"] == [[], []] and ctx["order"] == [0, 1]
    tm.append([b, a], [50, 51])                      # both leaves shared -> two new chunks
    ctx = tm.context()
    assert ctx["chunks"][0][4] == 2 and ctx["chunks"][1][4] == 2
    assert [len(p) for p in ctx["private"]] == [1, 1]
    assert ctx["order"] == [1, 0]                    # creation serial: b's chunk grew first


def test_partial_tail_duplicates_not_shared():
    tm = TreeModel(4, 64)
    tm.add_sequence([1, 2, 3, 4, 5, 6])
    _, m, new = tm.add_sequence([1, 2, 3, 4, 5, 6])
    assert m == 4 and len(new) == 1                  # partial chunk never shared (T1)
    ctx = tm.context()
    assert ctx["shared"] == [(0, 0, 1)]


def _invariants(tm, seqs):
    ctx = tm.context()
    order = ctx["order"]
    assert sorted(order) == sorted(seqs)
    row_of = ctx["row_of"]
    recs = {cid: (par, sp, ln, ref, i, j) for (cid, par, sp, ln, ref, ft, lt, i, j) in ctx["chunks"]}
    # reconstruction + contiguity + ref conservation
    cover = {cid: [] for cid in recs}
    for sid, toks in seqs.items():
        assert tm.tokens_of(sid) == toks
        path = tm.path_ids(sid)
        for k, cid in enumerate(path):
            par, sp, ln, ref, i, j = recs[cid]
            assert sp == k * tm.c
            assert ln == tm.c or k == len(path) - 1
            cover[cid].append(row_of[sid])
    for cid, rows in cover.items():
        par, sp, ln, ref, i, j = recs[cid]
        assert ref == len(rows)
        assert sorted(rows) == list(range(i, j + 1))   # contiguous
        if ref >= 2:
            assert ln == tm.c                          # shared chunks are full (T1)
    used, free, created, hwm, waste = tm.memory_stats()
    assert created == used + free and used == len(recs) and hwm >= used
    # waste ("at most c - 1 unused slots per sequence"): only a
    # sequence's last chunk can be partial and partial chunks are never shared
    # (T1), so the unused slots are exactly sum over sequences of (-len) mod c,
    # computed here from the token counts alone
    assert waste == sum((-len(toks)) % tm.c for toks in seqs.values())
    assert waste <= (tm.c - 1) * len(seqs)
    ids = [cid for cid in recs] + tm.free
    assert len(set(ids)) == len(ids)                   # no chunk both used and free


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_invariants_and_sharing(seed):
    rng = random.Random(seed)
    c = rng.choice([2, 4, 16])
    tm = TreeModel(c, 10_000)
    prompts = [[rng.randint(1, 30000) for _ in range(rng.randint(0, 5 * c))] for _ in range(3)]
    seqs = {}
    for op in range(400):
        r = rng.random()
        if r < 0.3 or not seqs:
            p = rng.choice(prompts)
            toks = p[:rng.randint(0, len(p))] + [rng.randint(1, 30000) for _ in range(rng.randint(1, 2 * c))]
            sid, m, _ = tm.add_sequence(toks)
            seqs[sid] = list(toks)
        elif r < 0.45:
            sid = rng.choice(sorted(seqs))
            tm.remove_sequence(sid)
            del seqs[sid]
        else:
            ids = rng.sample(sorted(seqs), rng.randint(1, len(seqs)))
            new = [rng.randint(1, 30000) for _ in ids]
            tm.append(ids, new)
            for s, t in zip(ids, new):
                seqs[s].append(t)
        _invariants(tm, seqs)
    # order-free sharing definition (random private/decode tokens: no ties)
    got = set()
    ctx = tm.context()
    members = {}
    for sid in seqs:
        for k, cid in enumerate(tm.path_ids(sid)):
            members.setdefault((k, cid), set()).add(sid)
    for (k, cid), mem in members.items():
        if len(mem) >= 2:
            got.add((k, frozenset(mem)))
    assert got == expected_sharing(seqs, c)


def test_export_format_fig2():
    text = fig2_model().export()
    lines = text.splitlines()
    assert lines[0] == "chunks:"
    assert lines[1] == "0 -1 0 4 3 1 4"
    assert "order: 0 1 2" in lines
    assert "shared: (0,0,2) (1,0,2) (2,0,2)" in lines
    assert lines[-1] == "alloc: 8 0 8 8"
