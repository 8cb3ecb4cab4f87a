"""Pins for oracle/attention.py (C1, C2) against things other than itself."""
import math
import os
import random

import numpy as np
import pytest
import torch

from oracle.attention import (attend_fp64, attend_heads_fp64, attention_weights, attn_chunk_first,
                              attn_reduce, attn_seq_first, default_scale, partial_attn)
from oracle.tree_model import TreeModel

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _brute(q, K, V, s):
    """Pure-Python triple loop: o_k = sum_t e_t V[t][k] / sum_t e_t."""
    L, d = len(K), len(q)
    w = [s * sum(q[k] * K[t][k] for k in range(d)) for t in range(L)]
    mx = max(w)
    e = [math.exp(x - mx) for x in w]
    tot = sum(e)
    return [sum(e[t] * V[t][k] for t in range(L)) / tot for k in range(d)]


def _gold():
    vals = {}
    with open(os.path.join(GOLD, "eqn_worked.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            k, *v = line.split()
            vals[k] = [float(x) for x in v]
    return vals


@pytest.mark.parametrize("seed", range(40))
def test_c1_vs_bruteforce(seed):
    rng = random.Random(seed)
    d, L = rng.randint(1, 4), rng.randint(1, 9)
    q = [rng.uniform(-3, 3) for _ in range(d)]
    K = [[rng.uniform(-3, 3) for _ in range(d)] for _ in range(L)]
    V = [[rng.uniform(-3, 3) for _ in range(d)] for _ in range(L)]
    s = rng.choice([1.0, default_scale(d), 0.37])
    np.testing.assert_allclose(attend_fp64(q, K, V, s), _brute(q, K, V, s), rtol=0, atol=1e-12)


@pytest.mark.parametrize("seed", range(10))
def test_c1_heads_vs_sdpa(seed):
    g = torch.Generator().manual_seed(seed)
    h, L, d = 3, 37, 16
    q = torch.randn(h, d, generator=g, dtype=torch.float64) * 4
    K = torch.randn(L, h, d, generator=g, dtype=torch.float64)
    V = torch.randn(L, h, d, generator=g, dtype=torch.float64)
    ref = torch.nn.functional.scaled_dot_product_attention(
        q[:, None, :], K.permute(1, 0, 2), V.permute(1, 0, 2))[:, 0, :]
    out = attend_heads_fp64(q.numpy(), K.numpy(), V.numpy(), default_scale(d))
    np.testing.assert_allclose(out, ref.numpy(), rtol=0, atol=1e-12)
    for hh in range(h):  # per-head C1 agrees with the batched form
        np.testing.assert_allclose(attend_fp64(q[hh], K[:, hh], V[:, hh], default_scale(d)),
                                   out[hh], rtol=0, atol=1e-13)


def test_c1_closed_forms():
    rng = np.random.default_rng(0)
    L, d = 13, 8
    V = rng.standard_normal((L, d))
    K = np.tile(rng.standard_normal(d), (L, 1))          # identical keys -> uniform weights
    q = rng.standard_normal(d)
    np.testing.assert_allclose(attend_fp64(q, K, V, 0.5), V.mean(axis=0), atol=1e-14)
    np.testing.assert_allclose(attend_fp64(q, np.zeros((L, d)), V, 0.5), V.mean(axis=0), atol=1e-14)
    np.testing.assert_allclose(attend_fp64(q, K[:1], V[:1], 0.5), V[0], atol=0)   # singleton
    w = attention_weights(q, rng.standard_normal((L, d)) * 5, 1.0)
    assert abs(w.sum() - 1.0) < 1e-15 and (w > 0).all()
    # one-hot V rows: output equals the weights themselves
    Kr = rng.standard_normal((L, 16))
    qr = rng.standard_normal(16)
    Vh = np.eye(L, 16)
    np.testing.assert_allclose(attend_fp64(qr, Kr, Vh, 0.25)[:L], attention_weights(qr, Kr, 0.25), atol=1e-15)


def test_worked_values():
    g = _gold()
    q = np.array(g["eqn1.q"])
    K = np.array(g["eqn1.K"]).reshape(2, 2)
    V = np.array(g["eqn1.V"]).reshape(2, 2)
    O, m, n = partial_attn(q[None], K, V, g["eqn1.scale"][0])
    assert round(m[0], 5) == g["eqn1.m"][0]
    assert round(n[0], 5) == g["eqn1.n"][0]
    assert [round(x, 5) for x in O[0]] == g["eqn1.O"]
    oa, ma, na = g["eqn2.A"]
    ob, mb, nb = g["eqn2.B"]
    o, m2, n2 = attn_reduce(np.array([ob]), mb, nb, np.array([oa]), ma, na)
    assert round(o[0], 5) == g["eqn2.O"][0]
    assert round(n2, 5) == g["eqn2.n"][0]
    assert round(o[0] / n2, 5) == g["eqn2.out"][0]
    # and it equals the direct softmax over logits {1, 0} with values that
    # reproduce the partial sums: o/n = (2*e^1*... ) -- check by re-basing
    direct = (oa * math.exp(ma) + ob * math.exp(mb)) / (na * math.exp(ma) + nb * math.exp(mb))
    assert abs(o[0] / n2 - direct) < 1e-14


def test_reduce_identity_and_guard():
    o0, m0, n0 = np.zeros(3), -np.inf, 0.0
    oc, mc, nc = np.array([1.0, 2.0, 3.0]), 0.3, 2.0
    o, m, n = attn_reduce(oc, mc, nc, o0, m0, n0)
    assert (o == oc).all() and m == mc and n == nc          # exact identity merge
    o, m, n = attn_reduce(o0, m0, n0, o0, m0, n0)           # empty + empty: no NaN
    assert m == -np.inf and n == 0.0 and not np.isnan(o).any()
    # reading A2: logits around -800 — the paper's literal (0,0,0) init underflows
    q = np.array([1.0])
    K = np.array([[-800.0], [-801.0]])
    V = np.array([[1.0], [3.0]])
    O, mm, nn = partial_attn(q[None], K, V, 1.0)
    o, m, n = attn_reduce(O[0], mm[0], nn[0], np.zeros(1), -np.inf, 0.0)
    np.testing.assert_allclose(o / n, attend_fp64(q, K, V, 1.0), atol=1e-14)
    o_lit, m_lit, n_lit = attn_reduce(O[0], mm[0], nn[0], np.zeros(1), 0.0, 0.0)
    with np.errstate(invalid="ignore"):
        assert np.isnan(o_lit / n_lit).all()


@pytest.mark.parametrize("seed", range(30))
def test_c2_partition_and_merge_order_invariance(seed):
    rng = np.random.default_rng(seed)
    L, d = int(rng.integers(1, 60)), int(rng.choice([4, 16]))
    alpha = float(rng.choice([1.0, 8.0, 30.0]))
    q = rng.standard_normal(d) * alpha
    K = rng.standard_normal((L, d))
    V = rng.standard_normal((L, d))
    s = default_scale(d)
    ref = attend_fp64(q, K, V, s)
    cuts = sorted(set(rng.integers(0, L + 1, size=int(rng.integers(0, 6))).tolist()) | {0, L})
    parts = [partial_attn(q[None], K[a:b], V[a:b], s) for a, b in zip(cuts[:-1], cuts[1:])]
    order = rng.permutation(len(parts))
    o, m, n = np.zeros(d), -np.inf, 0.0
    for k in order:
        O_c, m_c, n_c = parts[k]
        o, m, n = attn_reduce(O_c[0], m_c[0], n_c[0], o, m, n)
    np.testing.assert_allclose(o / n, ref, rtol=0, atol=1e-12)
    # tree-shaped merge: merge pairs, then merge the results
    accs = [(P[0][0], P[1][0], P[2][0]) for P in parts]
    while len(accs) > 1:
        nxt = []
        for a in range(0, len(accs), 2):
            if a + 1 < len(accs):
                nxt.append(attn_reduce(*accs[a], *accs[a + 1]))
            else:
                nxt.append(accs[a])
        accs = nxt
    o, m, n = accs[0]
    np.testing.assert_allclose(o / n, ref, rtol=0, atol=1e-12)


def _tree_case(seed):
    rng = random.Random(seed)
    c = rng.choice([2, 4, 8])
    tm = TreeModel(c, 10_000)
    prompt = [rng.randint(1, 50) for _ in range(rng.randint(0, 4 * c))]
    seqs = {}
    for _ in range(rng.randint(1, 6)):
        toks = prompt[:rng.randint(0, len(prompt))] + [rng.randint(1, 50) for _ in range(rng.randint(1, 3 * c))]
        sid, _, _ = tm.add_sequence(toks)
        seqs[sid] = toks
    for _ in range(rng.randint(0, c + 2)):
        ids = list(seqs)
        rng.shuffle(ids)
        new = [rng.randint(1, 50) for _ in ids]
        tm.append(ids, new)
        for s, t in zip(ids, new):
            seqs[s].append(t)
    return tm, seqs


@pytest.mark.parametrize("seed", range(25))
def test_alg1_alg2_equal_c1(seed):
    """Alg 1 + Alg 2 over the replay model's context equal C1 on every row."""
    tm, seqs = _tree_case(seed)
    d, h = 8, 1
    rng = np.random.default_rng(seed)
    kv = {}  # (token, pos) -> (k, v): KV depends only on token and position

    def kv_of(tok, pos):
        if (tok, pos) not in kv:
            kv[(tok, pos)] = (rng.standard_normal(d), rng.standard_normal(d))
        return kv[(tok, pos)]

    chunk_tokens = {}
    for sid, toks in seqs.items():
        assert tm.tokens_of(sid) == toks
    ctx = tm.context()
    chunks = {cid: (sp, ln) for (cid, par, sp, ln, ref, ft, lt, i, j) in ctx["chunks"]}
    # tokens of a chunk: read through any sequence whose path holds it
    for sid in seqs:
        toks = tm.tokens_of(sid)
        for cid in tm.path_ids(sid):
            sp, ln = chunks[cid]
            chunk_tokens[cid] = [(toks[p], p) for p in range(sp, sp + ln)]

    def chunk_kv(cid):
        pairs = chunk_tokens[cid]
        K = np.array([kv_of(t, p)[0] for t, p in pairs]).reshape(-1, d)
        V = np.array([kv_of(t, p)[1] for t, p in pairs]).reshape(-1, d)
        return K, V

    order = ctx["order"]
    Q = rng.standard_normal((len(order), d)) * 3
    s = default_scale(d)
    saved = attn_chunk_first(Q, ctx["shared"], chunk_kv, s)
    out = attn_seq_first(Q, ctx["shared"], ctx["private"], saved, chunk_kv, s)
    for r, sid in enumerate(order):
        toks = seqs[sid]
        K = np.array([kv_of(t, p)[0] for p, t in enumerate(toks)])
        V = np.array([kv_of(t, p)[1] for p, t in enumerate(toks)])
        np.testing.assert_allclose(out[r], attend_fp64(Q[r], K, V, s), rtol=0, atol=1e-12)
