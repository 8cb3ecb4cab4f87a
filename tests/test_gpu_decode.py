"""GPU parity of the one-launch decode step (chunkattn_append_attend, the K5
cluster decode kernel: append + chunk-first + seq-first + cluster merge in one
kernel) against the fp64 oracle, plus its bit-level invariants.  Tolerances as
test_gpu_parity.py (reading A11)."""
import random

import numpy as np
import pytest
import torch

import synth
from tests.gpu_workload import Harness, build_shared, decode_tokens

pytestmark = pytest.mark.gpu

TOL = {("f16", "f16"): 2e-3, ("bf16", "f32"): 2e-3, ("f16", "f32"): 2e-3, ("bf16", "bf16"): 4e-3}


def _case(seed):
    rng = random.Random(1000 + seed)
    dt, odt = rng.choice([("f16", "f16"), ("bf16", "f32")])
    c = rng.choice([16, 32, 64, 64, 64])
    d = rng.choice([64, 128])
    h = rng.choice([1, 2, 4])
    b = rng.randint(1, 12)
    return dict(dt=dt, odt=odt, c=c, d=d, h=h, b=b, alpha=rng.choice([1.0, 8.0]),
                mode=rng.choice(["chunk", "chunk", "chunk", "b0", "b1"]), n_shared=rng.randint(0, 4 * c),
                privates=[rng.randint(0, 3 * c) for _ in range(b)], steps=rng.randint(1, 4), rng=rng)


@pytest.mark.parametrize("opts", ["", "dk_cs=1", "dk_cs=3", "dk_max_rows=16", "dk_cs=16", "dk_umma=0",
                                  "dk_umma=2", "dk_umma=2,dk_cs=3", "dk_umma=2,dk_max_rows=16"])
@pytest.mark.parametrize("seed", range(40))
def test_append_attend_property_suite(seed, opts):
    """Random trees (shared prompt, private tails 0..3c incl. empty, 1..4 fused
    decode steps, permuted seq_ids order every step), cluster sizes auto / 1 /
    3 and 16-row blocks, chunk-first units on mma.sync (dk_umma=0) and on
    tcgen05 (dk_umma=2, c = 64 cases): every (row, head) against the oracle."""
    p = _case(seed)
    hs = Harness(p["h"], p["d"], p["c"], p["dt"], p["odt"], seed=seed, alpha=p["alpha"], mode=p["mode"], opts=opts)
    ids = build_shared(hs, p["n_shared"], p["privates"], seed_tag=seed)
    tol = TOL[(p["dt"], p["odt"])]
    hs.check(ids, tol)  # attend-only first (rows without a private chunk)
    for st in range(p["steps"]):
        hs.step = st + 1
        order = ids[:]
        p["rng"].shuffle(order)
        hs.append_attend(order, decode_tokens(hs, order), tol)
    hs.step += 1
    hs.check(ids, tol)  # attend-only on the lengths the fused steps left on the device


@pytest.mark.parametrize("dt,odt", [("f16", "f16"), ("bf16", "f32")])
def test_append_attend_matches_two_call_path_and_pool(dt, odt):
    """The fused step leaves the same pool bytes as append_kv (bit-exact K/V
    rows in their swizzled slots) and outputs within rounding of the two-call
    path; crossing a chunk boundary (structural step) included."""
    a = Harness(4, 128, 64, dt, odt, seed=5, alpha=8.0)
    b = Harness(4, 128, 64, dt, odt, seed=5, alpha=8.0, opts="dk=0")
    ia = build_shared(a, 128, [62, 63, 0, 5, 64])
    ib = build_shared(b, 128, [62, 63, 0, 5, 64])
    for st in range(1, 4):
        a.step = b.step = st
        toks = decode_tokens(a, ia)
        _, oa = a.append_attend(ia, toks, 2e-3)
        b.append(ib, toks)
        _, ob = b.attend(ib)
        assert float((oa.double() - ob.double()).abs().max()) <= 2e-3
    assert torch.equal(a.ca.k_pool, b.ca.k_pool) and torch.equal(a.ca.v_pool, b.ca.v_pool)


def test_append_attend_deterministic_and_layers():
    """Two handles fed the same steps give bitwise-equal outputs; two layers
    with identical K/V give bitwise-equal outputs per layer."""
    outs = []
    for _ in range(2):
        hs = Harness(8, 128, 64, "f16", "f16", seed=9, alpha=8.0)
        ids = build_shared(hs, 640, [3, 70, 0, 129, 1, 64])
        for st in range(1, 4):
            hs.step = st
            _, o = hs.append_attend(ids, decode_tokens(hs, ids), 2e-3)
        outs.append(o.clone())
    assert torch.equal(outs[0], outs[1])

    def kv2(which, toks, pos):  # identical K/V in both layers
        one = synth.kv_values(9, which, toks, pos, 1, 4, 64)
        return torch.cat([one, one], dim=1)

    hs = Harness(4, 64, 16, "f16", "f16", num_layers=2, seed=9, alpha=8.0, kv_fn=kv2)
    ids = build_shared(hs, 48, [5, 17, 0])
    for st in range(1, 4):
        hs.step = st
        toks = decode_tokens(hs, ids)
        pos = [len(hs.seqs[s]) for s in ids]
        k, v = hs.kv(toks, pos)
        for s, t in zip(ids, toks):
            hs.seqs[s].append(int(t))
        q = hs.queries(ids, 0).to(hs.dev, hs.dt).contiguous()
        o0 = hs.ca.append_attend(ids, toks, k[:, 0].to(hs.dev, hs.dt).contiguous(),
                                 v[:, 0].to(hs.dev, hs.dt).contiguous(), q, layer=0)
        o1 = hs.ca.append_attend(ids, None, k[:, 1].to(hs.dev, hs.dt).contiguous(),
                                 v[:, 1].to(hs.dev, hs.dt).contiguous(), q, layer=1)
        torch.cuda.synchronize()
        assert torch.equal(o0, o1)
        ref = hs.oracle(ids, hs.queries(ids, 0))
        assert float(np.abs(o0.double().cpu().numpy() - ref).max()) <= 2e-3


@pytest.mark.parametrize("umma", [0, 2])
@pytest.mark.parametrize("p", [1, 65])
def test_config2_append_attend_full_size(p, umma):
    """BASELINE configs[1] (b = 32, n_s = 2048, 32 x 128 fp16) through the
    fused step at completion tokens 1..3 after a p-1 token question, chunk-first
    units on mma.sync and on tcgen05: every row, every head against the oracle."""
    hs = Harness(32, 128, 64, "f16", "f16", seed=3, alpha=8.0, max_chunks=512, opts=f"dk_umma={umma}")
    ids = build_shared(hs, 2048, [p - 1] * 32)
    for st in range(1, 4):
        hs.step = st
        hs.append_attend(ids, decode_tokens(hs, ids), 2e-3, rows=list(range(32)) if st == 3 else [0, 17, 31])
    assert hs.ca.schedule_info()["dk_um"] == (1 if umma else 0)
