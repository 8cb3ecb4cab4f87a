"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded inputs.  Tolerances (north_star / DESIGN.md reading A11): 1e-5 for
fp32, 2e-3 max-abs for fp16 (fp16 out) and bf16 (fp32 out)."""
import random

import numpy as np
import pytest
import torch

import synth
from oracle.tree_model import TreeModel
from tests.gpu_workload import Harness, build_shared, decode_tokens

pytestmark = pytest.mark.gpu

TOL = {("f32", "f32"): 1e-5, ("f16", "f16"): 2e-3, ("bf16", "f32"): 2e-3, ("f16", "f32"): 2e-3}
# kernel variants exercised beside the default path (the K5 cluster decode
# kernel where the shape allows): the persistent fused kernel, the two-kernel
# phase pair (tcgen05 chunk-first where supported), with the mma.sync
# chunk-first kernel, and its 4-warp CTA (PDL co-residency)
VARIANTS = ["", "dk=0", "dk=0,fused=0", "dk=0,fused=0,cf_umma=0", "dk=0,fused=0,cf_umma=0,cf_small=1"]


# --------------------------------------------------------------- config 1 ---
@pytest.mark.parametrize("dt,odt", [("f32", "f32"), ("f16", "f16"), ("bf16", "f32")])
@pytest.mark.parametrize("mode", ["chunk", "b0", "b1"])
def test_tiny_config(dt, odt, mode):
    """BASELINE configs[0]: 4 seqs, 8 heads x 64, chunk 16, shared prompt 64 +
    {0, 1, 16, 32} private tokens; attend-only (a zero-private row) then one
    decode step (append, then attend)."""
    hs = Harness(8, 64, 16, dt, odt, seed=1, alpha=8.0, mode=mode)
    ids = build_shared(hs, 64, [0, 1, 16, 32])
    hs.check(ids, TOL[(dt, odt)])
    hs.step = 1
    hs.append(ids, decode_tokens(hs, ids))
    hs.check(ids, TOL[(dt, odt)])
    if mode == "chunk":
        assert "shared: (0,0,3) (1,0,3) (2,0,3) (3,0,3)" in hs.ca.export_context()


# ----------------------------------------------------------- property suite ---
def _random_case(seed):
    rng = random.Random(seed)
    dt, odt = rng.choice([("f32", "f32"), ("f16", "f16"), ("bf16", "f32")])
    c = rng.choice([16, 64] if dt != "f32" else [4, 16, 64])
    if rng.random() < 0.15:
        c = rng.choice([4, 8, 32])
    d = rng.choice([64, 128])
    h = rng.choice([1, 4])
    b = rng.randint(1, 8)
    alpha = rng.choice([1.0, 8.0])
    mode = rng.choice(["chunk", "chunk", "b0", "b1"])
    return dict(dt=dt, odt=odt, c=c, d=d, h=h, b=b, alpha=alpha, mode=mode,
                n_shared=rng.randint(0, 4 * c), privates=[rng.randint(0, 3 * c) for _ in range(b)],
                steps=rng.randint(0, 3), rng=rng)


@pytest.mark.parametrize("opts", VARIANTS)
@pytest.mark.parametrize("seed", range(60))
def test_property_suite(seed, opts):
    p = _random_case(seed)
    hs = Harness(p["h"], p["d"], p["c"], p["dt"], p["odt"], seed=seed, alpha=p["alpha"], mode=p["mode"], opts=opts)
    ids = build_shared(hs, p["n_shared"], p["privates"], seed_tag=seed)
    tol = TOL[(p["dt"], p["odt"])]
    hs.check(ids, tol)
    for st in range(p["steps"]):
        hs.step = st + 1
        hs.append(ids, decode_tokens(hs, ids))
        order = ids[:]
        p["rng"].shuffle(order)
        hs.check(order, tol)


# ---------------------------------------------------------------- config 2 ---
@pytest.mark.parametrize("opts", VARIANTS)
@pytest.mark.parametrize("p", [1, 65])
@pytest.mark.parametrize("dt,odt", [("f16", "f16"), ("bf16", "f32")])
def test_config2_llama_b32_s2048(p, dt, odt, opts):
    """BASELINE configs[1]: 32 heads x 128, fp16, chunk 64, batch 32, shared
    system prompt 2048; p private tokens (question p-1 + current token)."""
    hs = Harness(32, 128, 64, dt, odt, seed=3, alpha=8.0, max_chunks=512, opts=opts)
    ids = build_shared(hs, 2048, [p - 1] * 32)
    hs.step = 1
    hs.append(ids, decode_tokens(hs, ids))
    err, _ = hs.check(ids, TOL[(dt, odt)])
    ctr = hs.ca.counters()
    info = hs.ca.schedule_info()
    # the shared prompt runs as chunk-first work: partial slots (persistent
    # kernels) or chunk-first units in the K5 cluster schedule
    assert ctr["slots"] > 0 or (info["dk"] == 1 and info["dk_units"] >= 32 * info["dk_hg"])


@pytest.mark.parametrize("mode", ["b0", "b1"])
def test_config2_baselines(mode):
    hs = Harness(32, 128, 64, "f16", "f16", seed=3, alpha=8.0, max_chunks=2200, mode=mode)
    ids = build_shared(hs, 2048, [0] * 32)
    hs.step = 1
    hs.append(ids, decode_tokens(hs, ids))
    hs.check(ids, 2e-3, rows=list(range(0, 32, 5)))


# -------------------------------------------------------- invariant probes ---
def test_v_ones_gives_ones():
    def kv_fn(which, toks, pos):
        x = synth.kv_values(5, which, toks, pos, 1, 4, 128)
        return torch.ones_like(x) if which == synth.TID_V else x * 8
    hs = Harness(4, 128, 64, "f16", "f32", seed=5, alpha=8.0, kv_fn=kv_fn)
    ids = build_shared(hs, 256, [0, 3, 70, 200])
    _, out = hs.attend(ids)
    assert torch.allclose(out, torch.ones_like(out), atol=1e-6, rtol=0), float((out - 1).abs().max())


def test_one_hot_values_give_weights():
    """V row t = e_t (L <= d): the output is the softmax weights themselves."""
    def kv_fn(which, toks, pos):
        x = synth.kv_values(6, which, toks, pos, 1, 2, 128)
        if which == synth.TID_V:
            x = torch.zeros_like(x)
            for i, pp in enumerate(pos.tolist()):
                x[i, :, :, pp] = 1.0
        return x
    hs = Harness(2, 128, 16, "f32", "f32", seed=6, alpha=8.0, kv_fn=kv_fn)
    ids = build_shared(hs, 64, [0, 10, 40])
    q64, out = hs.attend(ids)
    from oracle.attention import attention_weights, default_scale
    for r, sid in enumerate(ids):
        toks = hs.seqs[sid]
        k, _ = hs.kv(toks, list(range(len(toks))))
        for head in range(2):
            w = attention_weights(q64[r, head].numpy(), k[:, 0, head].cpu().numpy(), default_scale(128))
            np.testing.assert_allclose(out[r, head, :len(toks)].cpu().numpy(), w, atol=1e-6)
            assert float(out[r, head, len(toks):].abs().max()) == 0.0


def test_large_logits_planted_keys():
    """|logit| ~ 77-106: keys planted as +-sign(q) on some tokens."""
    qseed = 7
    qv = synth.q_values(qseed, torch.arange(64), 0, 1, 2, 128, alpha=16.0)

    def kv_fn(which, toks, pos):
        x = synth.kv_values(qseed, which, toks, pos, 1, 2, 128)
        if which == synth.TID_K:
            planted = (toks % 7 == 0)
            sgn = torch.sign(qv[0, 0])[None, None, :]
            x[planted] = torch.where(pos[planted, None, None, None] % 2 == 0, 1.0, -1.0) * sgn
        return x
    hs = Harness(2, 128, 64, "f16", "f16", seed=qseed, alpha=16.0, kv_fn=kv_fn)
    ids = build_shared(hs, 320, [5, 64, 100])
    q64, out = hs.attend(ids)
    ref = hs.oracle(ids, q64)
    assert np.isfinite(out.float().cpu().numpy()).all()
    assert float(np.abs(out.double().cpu().numpy() - ref).max()) <= 2e-3


def test_shared_vs_unshared_and_b1_agree():
    outs = {}
    for mode in ["chunk", "b0", "b1"]:
        hs = Harness(4, 128, 64, "f16", "f32", seed=9, alpha=8.0, mode=mode)
        ids = build_shared(hs, 640, [1, 33, 64, 130, 7])
        outs[mode] = hs.attend(ids)[1].double().cpu()
    assert float((outs["chunk"] - outs["b0"]).abs().max()) <= 2e-3
    assert float((outs["chunk"] - outs["b1"]).abs().max()) <= 2e-3


# ------------------------------------------------ determinism / scheduling ---
def test_determinism_permutation_idempotence():
    hs = Harness(8, 128, 64, "f16", "f16", seed=11, alpha=8.0)
    ids = build_shared(hs, 1024, [3, 70, 0, 129, 64, 9, 1, 250])
    q64 = hs.queries(ids)
    q = q64.to(hs.dev, hs.dt)
    o1 = hs.ca.attend(ids, q).clone()
    up = hs.ca.counters()["uploads"]
    o2 = hs.ca.attend(ids, q).clone()
    assert torch.equal(o1, o2)
    assert hs.ca.counters()["uploads"] == up          # idempotent call uploads nothing
    perm = [5, 2, 7, 0, 1, 6, 3, 4]
    o3 = hs.ca.attend([ids[i] for i in perm], q[perm].contiguous())
    assert torch.equal(o3, o1[perm])                  # permutation permutes outputs bitwise
    hs2 = Harness(8, 128, 64, "f16", "f16", seed=11, alpha=8.0)
    ids2 = build_shared(hs2, 1024, [3, 70, 0, 129, 64, 9, 1, 250])
    assert torch.equal(hs2.ca.attend(ids2, q), o1)    # run-to-run reproducible
    assert hs2.ca.export_context() == hs.ca.export_context()


@pytest.mark.parametrize("dt,odt", [("f16", "f16"), ("bf16", "f32")])
def test_split_invariance_and_simt_chunk_first(dt, odt):
    hs = Harness(4, 128, 64, dt, odt, seed=13, alpha=8.0, opts="dk=0")
    ids = build_shared(hs, 2048, [2, 40, 65, 1, 0, 77, 128, 5, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18])
    q64 = hs.queries(ids)
    ref = hs.oracle(ids, q64)
    q = q64.to(hs.dev, hs.dt)
    for opt, val in [("cf_splits", 1), ("cf_splits", 2), ("cf_splits", 4), ("cf_splits", 32), ("cf_splits", 0),
                     ("cf_simt", 1), ("sf_simt", 1), ("sf_ctas", 1), ("sf_ctas", 7), ("sf_ctas", 333),
                     ("sf_ctas", 2048)]:
        hs.ca.set_option(opt, val)
        o1 = hs.ca.attend(ids, q).clone()
        o2 = hs.ca.attend(ids, q).clone()
        assert torch.equal(o1, o2)                   # each fixed schedule is bitwise reproducible
        err = float(np.abs(o1.double().cpu().numpy() - ref).max())
        assert err <= 2e-3, (opt, val, err)
        if opt in ("cf_simt", "sf_simt"):
            hs.ca.set_option(opt, 0)


@pytest.mark.parametrize("c,opts", [(16, ""), (64, ""), (64, "dk=0"), (64, "dk=0,fused=0")])
def test_layers_independent(c, opts):
    """Two layers share one tree; each layer's attention reads its own pool
    slice (c = 64 with fused=0: the tcgen05 chunk-first's TMA row offset)."""
    hs = Harness(4, 64, c, "f16", "f16", num_layers=2, seed=15, alpha=8.0, opts=opts)
    ids = build_shared(hs, 3 * c, [0, 5, c + 20])
    for layer in (0, 1):
        hs.check(ids, 2e-3, layer=layer)


# ----------------------------------------------------------- tree on GPU ---
def test_pool_contents_match_supplied_kv():
    hs = Harness(2, 64, 16, "bf16", "f32", seed=17, max_chunks=64)
    tm = TreeModel(16, 64)
    ids = build_shared(hs, 40, [3, 17, 0])
    for sid in ids:
        tm.add_sequence(hs.seqs[sid])
    hs.step = 1
    toks = decode_tokens(hs, ids)
    hs.append(ids, toks)
    tm.append(ids, toks)
    assert hs.ca.export_context() == tm.export()
    torch.cuda.synchronize()
    kp = hs.ca.k_pool.cpu()
    vp = hs.ca.v_pool.cpu()
    idx = torch.arange(64)

    def unswz(row, s):  # 16-byte groups (8 x 16-bit) of slot s are XOR-permuted by s % 8
        return row[:, ((idx // 8) ^ (s & 7)) * 8 + idx % 8]
    for sid in ids:
        k, v = hs.kv(hs.seqs[sid], list(range(len(hs.seqs[sid]))))
        slots = tm.token_slots(sid)
        gk = torch.stack([unswz(kp[0, c, :, s, :], s) for c, s in slots]).double()
        gv = torch.stack([unswz(vp[0, c, :, s, :], s) for c, s in slots]).double()
        assert torch.equal(gk, k[:, 0].cpu()) and torch.equal(gv, v[:, 0].cpu())


def test_edge_cases_and_reuse():
    hs = Harness(4, 128, 64, "f16", "f16", seed=19, alpha=8.0, max_chunks=40)
    # b = 1: no chunk-first work at all
    a, _ = hs.add(synth.token_ids(19, 1, 1, 130).tolist())
    hs.check([a], 2e-3)
    # full duplicate of an exact multiple of c: a zero-private row (attend-only)
    base = synth.token_ids(19, 1, 2, 128).tolist()
    b, m = hs.add(base)
    c, m2 = hs.add(base)
    assert m == 0 and m2 == 128
    hs.check([a, b, c], 2e-3)
    # last chunk lengths 1, c-1, c
    d1, _ = hs.add(base + [5])
    d2, _ = hs.add(base + synth.token_ids(19, 1, 3, 63).tolist())
    hs.check([a, b, c, d1, d2], 2e-3)
    # removes then reuse of released chunks (stale tails must be masked)
    hs.remove(a)
    hs.remove(d2)
    e, _ = hs.add(synth.token_ids(19, 1, 4, 70).tolist())
    ids = [b, c, d1, e]
    hs.check(ids, 2e-3)
    for st in range(3):
        hs.step = st + 1
        hs.append(ids, decode_tokens(hs, ids))
        hs.check(ids, 2e-3)
    # capacity exhaustion rolls back and leaves the cache usable
    before = hs.ca.export_context()
    with pytest.raises(Exception):
        hs.add(synth.token_ids(19, 1, 5, 64 * 40).tolist())
    assert hs.ca.export_context() == before
    hs.check(ids, 2e-3)


@pytest.mark.parametrize("opts", VARIANTS)
def test_two_level_tree_decode_evict(opts):
    """Small version of BASELINE configs[3]: system prompt + per-group examples,
    decode with eviction/replacement; parity and byte-exact tables at checkpoints."""
    rng = random.Random(21)
    c = 16
    hs = Harness(4, 64, c, "f16", "f16", seed=21, alpha=8.0, max_chunks=600, opts=opts)
    tm = TreeModel(c, 600)
    sys_p = synth.token_ids(21, synth.TAG_SYS, 0, 64).tolist()
    groups = [synth.token_ids(21, synth.TAG_GROUP, g, 64).tolist() for g in range(4)]
    live, target, k = [], {}, 0

    def spawn():
        nonlocal k
        g = rng.randrange(4)
        q = synth.token_ids(21, synth.TAG_PRIV, k, rng.randint(1, c - 1)).tolist()
        k += 1
        toks = sys_p + groups[g] + q
        sid, _ = hs.add(toks)
        tm.add_sequence(toks)
        live.append(sid)
        target[sid] = rng.randint(8, 60)
    for _ in range(16):
        spawn()
    for step in range(1, 90):
        hs.step = step
        toks = decode_tokens(hs, live)
        hs.append(live, toks)
        tm.append(live, toks)
        for sid in list(live):
            target[sid] -= 1
            if target[sid] == 0:
                hs.remove(sid)
                tm.remove_sequence(sid)
                live.remove(sid)
                spawn()
        if step in (1, 15, 16, 40, 89):
            assert hs.ca.export_context() == tm.export()
            hs.check(live, 2e-3)
    for sid in list(live):
        hs.remove(sid)
        tm.remove_sequence(sid)
    st = hs.ca.memory_stats()
    assert st["used"] == 0 and st["free"] == st["created"]


def test_head_sharded_handles_match_single_gpu():
    """Two head-slice handles on one GPU (what two ranks hold) concatenate to the
    single-handle output (the chunk-first split is forced equal; the seq-first
    CTA ranges differ with the head count, so agreement is within rounding)."""
    H, d, c, seed = 8, 128, 64, 23
    full = Harness(H, d, c, "f16", "f16", seed=seed, alpha=8.0, opts="dk=0")
    ids = build_shared(full, 640, [3, 70, 0, 129])
    halves = []
    for h0 in (0, 4):
        def kv_fn(which, toks, pos, h0=h0):
            return synth.kv_values(seed, which, toks, pos, 1, 4, d, head_offset=h0)
        hs = Harness(4, d, c, "f16", "f16", seed=seed, alpha=8.0, kv_fn=kv_fn, opts="dk=0")
        build_shared(hs, 640, [3, 70, 0, 129])
        halves.append(hs)
    q64 = full.queries(ids)
    for opt in (("cf_splits", 2), ("sf_ctas", 16)):
        full.ca.set_option(*opt)
        for hs in halves:
            hs.ca.set_option(*opt)
    ref = full.ca.attend(ids, q64.to(full.dev, full.dt).contiguous())
    parts = [hs.ca.attend(ids, q64[:, i * 4:(i + 1) * 4].to(hs.dev, hs.dt).contiguous()) for i, hs in enumerate(halves)]
    assert float((torch.cat(parts, dim=1).double() - ref.double()).abs().max()) <= 1e-3


def test_host_buffers_zero_copy_match_device():
    """The C ABI takes pinned host q / k / v / out (UVA): the kernels read and
    write them over PCIe; results are bitwise those of device buffers."""
    import numpy as _np
    outs = []
    for host in (False, True):
        hs = Harness(4, 128, 64, "f16", "f16", seed=23, alpha=8.0)
        ids = build_shared(hs, 256, [0, 3, 70, 130, 5])
        n = len(ids)
        ida = _np.asarray(ids, dtype=_np.int64)
        stream = torch.cuda.current_stream().cuda_stream
        res = []
        for st in range(3):
            hs.step = st + 1
            toks = decode_tokens(hs, ids)
            pos = [len(hs.seqs[s]) for s in ids]
            k, v = hs.kv(toks, pos)
            for s, t in zip(ids, toks):
                hs.seqs[s].append(int(t))
            q = hs.queries(ids).to(torch.float16)
            k, v = k.to(torch.float16).contiguous(), v.to(torch.float16).contiguous()
            if host:
                k, v, q = k.cpu().pin_memory(), v.cpu().pin_memory(), q.cpu().pin_memory()
                out = torch.empty((n, 4, 128), dtype=torch.float16).pin_memory()
            else:
                k, v, q = k.cuda(), v.cuda(), q.cuda()
                out = torch.empty((n, 4, 128), dtype=torch.float16, device="cuda")
            hs.ca.append_raw(ida, _np.asarray(toks, dtype=_np.int32), k.data_ptr(), v.data_ptr(), stream)
            hs.ca.attend_raw(0, ida, q.data_ptr(), out.data_ptr(), stream)
            torch.cuda.synchronize()
            res.append(out.cpu().clone())
        outs.append(torch.stack(res))
        ref = hs.oracle(ids, hs.queries(ids))
        assert float(_np.abs(outs[-1][-1].double().numpy() - ref).max()) <= 2e-3
    assert torch.equal(outs[0], outs[1])


def test_decode_step_host_matches_device_path():
    """chunkattn_decode_step_host (host buffers, copies inside the call) gives
    bitwise the outputs of append_kv + attend on device buffers."""
    import numpy as _np
    outs = []
    for via_host in (False, True):
        hs = Harness(4, 128, 64, "f16", "f16", seed=29, alpha=8.0)
        ids = build_shared(hs, 192, [1, 64, 0, 90])
        n = len(ids)
        ida = _np.asarray(ids, dtype=_np.int64)
        staging = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
        res = []
        for st in range(3):
            hs.step = st + 1
            toks = decode_tokens(hs, ids)
            pos = [len(hs.seqs[s]) for s in ids]
            k, v = hs.kv(toks, pos)
            for s, t in zip(ids, toks):
                hs.seqs[s].append(int(t))
            q = hs.queries(ids).to(torch.float16)
            k, v = k.to(torch.float16).cpu(), v.to(torch.float16).cpu()
            if via_host:
                packed = torch.cat([q.reshape(-1), k.reshape(-1), v.reshape(-1)]).pin_memory()
                out = torch.empty((n, 4, 128), dtype=torch.float16).pin_memory()
                hs.ca.decode_step_host(ida, _np.asarray(toks, dtype=_np.int32), packed, out, staging)
            else:
                out = torch.empty((n, 4, 128), dtype=torch.float16, device="cuda")
                stream = torch.cuda.current_stream().cuda_stream
                kd, vd, qd = k.cuda(), v.cuda(), q.cuda()
                hs.ca.append_raw(ida, _np.asarray(toks, dtype=_np.int32), kd.data_ptr(), vd.data_ptr(), stream)
                hs.ca.attend_raw(0, ida, qd.data_ptr(), out.data_ptr(), stream)
            torch.cuda.synchronize()
            res.append(out.cpu().clone())
        outs.append(torch.stack(res))
        ref = hs.oracle(ids, hs.queries(ids))
        assert float(_np.abs(outs[-1][-1].double().numpy() - ref).max()) <= 2e-3
    assert torch.equal(outs[0], outs[1])
    with pytest.raises(Exception):  # staging too small
        hs.ca.decode_step_host(ida, _np.zeros(len(ids), dtype=_np.int32), torch.zeros(16).pin_memory(),
                               torch.zeros(16).pin_memory(), torch.empty(16, dtype=torch.uint8, device="cuda"))


# ------------------------------------------------- tcgen05 chunk-first (f3) ---
@pytest.mark.parametrize("d,c,dt,odt", [(128, 64, "f16", "f16"), (64, 64, "bf16", "f32"), (128, 128, "f16", "f32")])
def test_tcgen05_chunk_first_wide_runs(d, c, dt, odt):
    """Runs wider than the fused tile (130 and 70 rows) take the two-kernel
    schedule with the tcgen05 chunk-first (c = 64; c = 128 takes the mma.sync
    kernel): two row tiles per run, both head dims, a two-level tree (system prompt shared by
    all rows + a group prefix shared by 70), partial private chunks."""
    hs = Harness(2, d, c, dt, odt, seed=11, alpha=8.0, max_chunks=1024, opts="dk=0")
    sys_p = synth.token_ids(11, synth.TAG_SYS, 0, 3 * c).tolist()
    grp = synth.token_ids(11, synth.TAG_SYS, 1, c).tolist()
    ids = []
    for i in range(130):
        pre = sys_p + (grp if i < 70 else [])
        ids.append(hs.add(pre + synth.token_ids(11, synth.TAG_PRIV, i, i % 37).tolist())[0])
    hs.step = 1
    hs.append(ids, decode_tokens(hs, ids))
    hs.check(ids, TOL[(dt, odt)])
    for opts in ("dk=0,cf_umma=0", "dk=2"):  # the mma.sync chunk-first, then K5 forced (three row blocks), same tree
        hs2 = Harness(2, d, c, dt, odt, seed=11, alpha=8.0, max_chunks=1024, opts=opts)
        for i in range(130):
            pre = sys_p + (grp if i < 70 else [])
            hs2.add(pre + synth.token_ids(11, synth.TAG_PRIV, i, i % 37).tolist())
        hs2.step = 1
        hs2.append(ids, decode_tokens(hs2, ids))
        hs2.check(ids, TOL[(dt, odt)])


# ------------------------------------------- full-size shapes of the bench ---
@pytest.mark.parametrize("opts", ["", "dk=0", "dk=0,fused=0"])
def test_config2_full_size_last_timed_step(opts):
    """bench.py's workload at its largest timed step: b = 32, n_s = 2048, 512
    private tokens (context 2560), 32 x 128 fp16 -- every row, sampled heads
    checked against the fp64 oracle."""
    hs = Harness(32, 128, 64, "f16", "f16", seed=0, alpha=8.0, max_chunks=640, opts=opts)
    ids = build_shared(hs, 2048, [511] * 32)
    hs.step = 1
    hs.append(ids, decode_tokens(hs, ids))
    hs.check(ids, 2e-3, rows=list(range(0, 32, 3)))


@pytest.mark.parametrize("opts", ["", "dk=2"])
def test_config5_full_size_sampled_rows(opts):
    """BASELINE configs[4] on one GPU: b = 256, shared prompt 4096, 64-token
    private question + the decode token (auto: the 256-row run takes the
    two-kernel schedule with the tcgen05 chunk-first; dk=2: K5 forced, four
    64-row blocks): sampled rows against the fp64 oracle."""
    hs = Harness(32, 128, 64, "f16", "f16", seed=2, alpha=8.0, max_chunks=64 + 256 * 2 + 16, opts=opts)
    ids = build_shared(hs, 4096, [64] * 256)
    hs.step = 1
    hs.append(ids, decode_tokens(hs, ids))
    hs.check(ids, 2e-3, rows=[0, 1, 63, 127, 128, 200, 255])
