"""GPU parity of prefill attention with prefix lookup (SURVEY §8 row f1,
chunkattn_prefill_attend) against the fp64 oracle C4 (oracle/prefill.py):
sequences whose prompts match cached chunks only supply K/V (and queries) for
their unmatched suffix; every suffix query attends causally over the whole
sequence (shared chunks + own).  Tolerance 2e-3 max-abs (north_star)."""
import numpy as np
import pytest
import torch

import synth
from oracle.attention import default_scale
from oracle.prefill import causal_prefill_fp64
from tests.gpu_workload import Harness

pytestmark = pytest.mark.gpu


def _queries(seed, n, h, d):
    g = torch.Generator().manual_seed(seed)
    return torch.randn((n, h, d), generator=g, dtype=torch.float64) * 2.0


def _run(h, d, c, dt, odt, prompts, seed=0, opts=""):
    hs = Harness(h, d, c, dt, odt, seed=seed, alpha=8.0, opts=opts)
    ids, firsts = [], []
    for toks in prompts:
        m = hs.ca.match_prefix(toks)
        sid, matched = hs.add(toks, kv_first_pos=m)
        assert matched == m
        ids.append(sid)
        firsts.append(m)
    nq = sum(len(t) - f for t, f in zip(prompts, firsts))
    q = _queries(seed + 1, nq, h, d)
    out = hs.ca.prefill_attend(ids, firsts, q.to(hs.dev, hs.dt).contiguous())
    torch.cuda.synchronize()
    got = out.double().cpu().numpy()
    qr = q.to(hs.dt).double().numpy()  # the oracle sees the rounded queries
    err, row = 0.0, 0
    for toks, f in zip(prompts, firsts):
        K, V = hs.kv(toks, list(range(len(toks))))
        K = K.to(hs.dt).double().cpu().numpy()[:, 0]
        V = V.to(hs.dt).double().cpu().numpy()[:, 0]
        n = len(toks) - f
        ref = causal_prefill_fp64(qr[row:row + n], K, V, f, default_scale(d))
        err = max(err, float(np.abs(got[row:row + n] - ref).max()))
        row += n
    return err, firsts


# c = 64 takes the tcgen05 kernel (128-query tiles), other chunk sizes and
# cf_umma=0 the mma.sync kernel (64-query tiles)
@pytest.mark.parametrize("h,d,c,dt,odt,opts", [(4, 128, 64, "f16", "f16", ""), (4, 128, 64, "f16", "f16", "cf_umma=0"),
                                               (2, 64, 64, "bf16", "f32", ""), (2, 64, 16, "bf16", "f32", ""),
                                               (2, 128, 32, "f16", "f32", "")])
def test_prefill_with_prefix_lookup(h, d, c, dt, odt, opts):
    sys_prompt = synth.token_ids(3, synth.TAG_SYS, 0, 3 * c + 5).tolist()
    prompts = [
        sys_prompt + synth.token_ids(3, synth.TAG_PRIV, 0, 2 * c + 7).tolist(),   # first: full causal prefill
        sys_prompt + synth.token_ids(3, synth.TAG_PRIV, 1, 70).tolist(),          # matches 3 chunks
        sys_prompt[:c + 3] + synth.token_ids(3, synth.TAG_PRIV, 2, 5).tolist(),   # matches 1 chunk
        sys_prompt[:2 * c] + [11],                                                # two full chunks matched, one query
    ]
    err, firsts = _run(h, d, c, dt, odt, prompts, opts=opts)
    assert firsts[0] == 0 and firsts[1] == 3 * c and firsts[2] == c
    assert err <= 2e-3, err


@pytest.mark.parametrize("opts", ["", "cf_umma=0"])
def test_prefill_many_tiles_and_ragged_tail(opts):
    """A 700-token prompt (6 / 11 query tiles, ragged last tile and chunk), then
    two sequences that reuse 10 of its chunks."""
    c = 64
    base = synth.token_ids(5, synth.TAG_SYS, 0, 700).tolist()
    prompts = [base, base[:650] + [7, 8, 9], base[:640] + synth.token_ids(5, synth.TAG_PRIV, 1, 129).tolist()]
    err, firsts = _run(2, 128, c, "f16", "f16", prompts, seed=5, opts=opts)
    assert firsts == [0, 640, 640]
    assert err <= 2e-3, err


def test_prefill_empty_and_errors():
    hs = Harness(2, 128, 64, "f16", "f16")
    sid, _ = hs.add(list(range(1, 100)))
    q = torch.zeros((0, 2, 128), dtype=torch.float16, device=hs.dev)
    hs.ca.prefill_attend([sid], [99], q)  # no queries: nothing launched
    with pytest.raises(Exception):
        hs.ca.prefill_attend([sid], [100], q)  # first_pos past the end
    with pytest.raises(Exception):
        hs.ca.prefill_attend([sid + 7], [0], torch.zeros((99, 2, 128), dtype=torch.float16, device=hs.dev))


def test_prefill_second_layer():
    """prefill_attend on layer 1 of a two-layer pool (tcgen05 kernel, c = 64)."""
    from oracle.prefill import causal_prefill_fp64 as ref_fn
    hs = Harness(2, 128, 64, "f16", "f16", num_layers=2, seed=9, alpha=8.0)
    toks = synth.token_ids(9, synth.TAG_SYS, 0, 150).tolist()
    sid, _ = hs.add(toks)
    q = _queries(10, len(toks), 2, 128)
    out = hs.ca.prefill_attend([sid], [0], q.to(hs.dev, hs.dt).contiguous(), layer=1)
    torch.cuda.synchronize()
    K, V = hs.kv(toks, list(range(len(toks))))
    ref = ref_fn(q.to(hs.dt).double().numpy(), K.to(hs.dt).double().cpu().numpy()[:, 1],
                 V.to(hs.dt).double().cpu().numpy()[:, 1], 0, default_scale(128))
    assert float(np.abs(out.double().cpu().numpy() - ref).max()) <= 2e-3
