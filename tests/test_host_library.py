"""Host logic of the C-ABI library (no GPU): the library loads and exports every
symbol of include/chunkattn.h, and the C++ prefix tree / context builder
reproduces the replay oracle (oracle/tree_model.py) byte for byte."""
import ctypes
import random

import pytest

from oracle.tree_model import PoolExhausted, TreeModel
from paper_2402_15220_b200 import ChunkAttention, ChunkAttnError
from paper_2402_15220_b200 import _capi as C


def test_library_exports_header_symbols():
    syms = C.header_symbols()
    assert len(syms) >= 15
    L = C.lib()
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(C._SIGS)


def test_workspace_bytes_and_bad_config():
    cfg = C.Config(32, 128, 64, 1, C.CA_F16, C.CA_F16, 2, 1, 0.0, -1, 1000, 32, 4096)
    assert C.lib().chunkattn_workspace_bytes(ctypes.byref(cfg)) > 0
    bad = C.Config(32, 100, 64, 1, C.CA_F16, C.CA_F16, 2, 1, 0.0, -1, 1000, 32, 4096)
    assert C.lib().chunkattn_workspace_bytes(ctypes.byref(bad)) == 0
    with pytest.raises(ChunkAttnError):
        ChunkAttention(32, 100, 64, 1000, 32, 4096, device=None)


def _host(c, max_chunks, **kw):
    return ChunkAttention(4, 64, c, max_chunks, 256, 4096, device=None, **kw)


def test_fig2_byte_exact():
    ca = _host(4, 64)
    tm = TreeModel(4, 64)
    s0 = list(range(1, 17))
    for toks in (s0, s0[:12] + [101, 102, 103, 104], s0[:12] + [201, 202, 203, 204]):
        assert ca.add_sequence(toks) == tm.add_sequence(toks)[:2]
    ca.append_kv([1, 2], [900, 901])
    tm.append([1, 2], [900, 901])
    assert ca.export_context() == tm.export()
    assert "tuples: (0,0,2) (1,0,2) (2,0,2) (3,0,0) (4,1,1) (6,1,1) (5,2,2) (7,2,2)" in ca.export_context()
    assert ca.batch_order() == [0, 1, 2]


def _fuzz(seed, n_ops, c, max_chunks, threshold=2, prefix_match=True, check_every=1):
    rng = random.Random(seed)
    ca = _host(c, max_chunks, share_threshold=threshold, prefix_match=prefix_match)
    tm = TreeModel(c, max_chunks, share_threshold=threshold, prefix_match=prefix_match)
    prompts = [[rng.randint(1, 30000) for _ in range(rng.randint(0, 6 * c))] for _ in range(4)]
    live = []
    for op in range(n_ops):
        r = rng.random()
        if r < 0.25 or not live:
            p = rng.choice(prompts)
            if rng.random() < 0.1 and live:   # full duplicate of a live prompt prefix
                toks = p[:rng.randint(1, len(p))] if p else [7]
            else:
                toks = p[:rng.randint(0, len(p))] + [rng.randint(1, 30000) for _ in range(rng.randint(1, 2 * c))]
            if not toks:
                toks = [5]
            assert ca.match_prefix(toks) == tm.match_prefix(toks)
            try:
                exp = tm.add_sequence(toks)[:2]
            except PoolExhausted:
                with pytest.raises(ChunkAttnError) as ei:
                    ca.add_sequence(toks)
                assert ei.value.status == C.CA_ENOMEM
            else:
                assert ca.add_sequence(toks) == exp
                live.append(exp[0])
        elif r < 0.4:
            sid = rng.choice(live)
            assert ca.remove_sequence(sid) == len(tm.remove_sequence(sid))
            live.remove(sid)
        else:
            ids = rng.sample(live, rng.randint(1, len(live)))
            if rng.random() < 0.2:   # identical decode tokens -> decode-filled duplicate siblings
                toks = [42] * len(ids)
            else:
                toks = [rng.randint(1, 30000) for _ in ids]
            try:
                tm.append(ids, toks)
            except PoolExhausted:
                with pytest.raises(ChunkAttnError) as ei:
                    ca.append_kv(ids, toks)
                assert ei.value.status == C.CA_ENOMEM
            else:
                ca.append_kv(ids, toks)
        if op % check_every == 0:
            assert ca.export_context() == tm.export(), f"op {op}"
            st = ca.memory_stats()
            assert (st["used"], st["free"], st["created"], st["hwm"], st["waste_slots"]) == tm.memory_stats()
    assert ca.export_context() == tm.export()
    assert ca.batch_order() == tm.batch_order()
    return ca, tm, live


@pytest.mark.parametrize("seed", range(6))
def test_fuzz_byte_exact(seed):
    c = [4, 16, 64, 2, 8, 4][seed]
    _fuzz(seed, 1700, c, max_chunks=[300, 200, 60, 2000, 400, 40][seed])


def test_fuzz_baselines_modes():
    _fuzz(11, 600, 4, 500, threshold=1 << 30)        # B1: shared chunks walked per row
    _fuzz(12, 600, 4, 2000, prefix_match=False)      # B0: no sharing at all


def test_attend_validation_host_only():
    ca = _host(4, 64)
    a, _ = ca.add_sequence([1, 2, 3, 4, 5])
    b, _ = ca.add_sequence([1, 2, 3, 4, 6])
    ca.attend([a, b])                     # host-only: validates and builds the context
    ca.attend([b, a])
    with pytest.raises(ChunkAttnError) as ei:
        ca.attend([a])
    assert ei.value.status == C.CA_ESTATE
    with pytest.raises(ChunkAttnError) as ei:
        ca.attend([a, a])
    assert ei.value.status == C.CA_ESTATE
    with pytest.raises(ChunkAttnError) as ei:
        ca.attend([a, 99])
    assert ei.value.status == C.CA_ENOSEQ
    with pytest.raises(ChunkAttnError) as ei:
        ca.remove_sequence(99)
    assert ei.value.status == C.CA_ENOSEQ
    with pytest.raises(ChunkAttnError) as ei:
        ca.append_kv([a, a], [1, 2])
    assert ei.value.status == C.CA_EINVAL
    with pytest.raises(ChunkAttnError):
        ca.add_sequence([])
    with pytest.raises(ChunkAttnError) as ei:
        ca.attend([a, b], layer=3)
    assert ei.value.status == C.CA_EINVAL


def test_lazy_context_counters():
    """Context builds happen only on the paper's three triggers."""
    ca = _host(4, 64)
    ids = [ca.add_sequence([1, 2, 3, 4, 9 + k])[0] for k in range(3)]
    ca.attend(ids)
    b0 = ca.counters()["builds"]
    ca.attend(ids)
    assert ca.counters()["builds"] == b0            # no mutation: cached
    ca.append_kv(ids, [5, 6, 7])                    # slots 1 of the private leaves: no structural change
    ca.attend(ids)
    assert ca.counters()["builds"] == b0
    ca.append_kv(ids, [5, 6, 7])
    ca.append_kv(ids, [5, 6, 7])
    ca.attend(ids)
    assert ca.counters()["builds"] == b0
    ca.append_kv(ids, [5, 6, 7])                    # leaves full -> grow ("chunk full" trigger)
    assert ca.counters()["builds"] == b0 + 1
    ca.remove_sequence(ids[0])                      # "completed sequence leaving"
    ca.attend(ids[1:])
    assert ca.counters()["builds"] == b0 + 2


def test_configs_whose_stages_do_not_fit_are_rejected():
    """ADVICE: two K/V tile stages of the persistent seq-first kernel must fit
    the 227 KB shared-memory limit -- f32 with chunk 128 x d 128 or 16-bit
    with chunk 256 x d 128 are rejected at creation (CA_EINVAL), not at the
    first attend."""
    import torch
    for dt, c in ((torch.float32, 128), (torch.float16, 256)):
        with pytest.raises(C.ChunkAttnError):
            ChunkAttention(4, 128, c, 64, 8, 1024, dtype=dt, device=None)
    ChunkAttention(4, 128, 64, 64, 8, 1024, dtype=torch.float32, device=None)  # fits


@pytest.mark.parametrize("question,umma,expect", [(0, 1, 1), (0, 0, 0), (0, 2, 1), (511, 1, 0), (511, 2, 1)])
def test_k5_tcgen05_variant_selection(question, umma, expect):
    """The K5 step takes the tcgen05 chunk-first variant (schedule_info
    "dk_um") when the step's chunk-first units are at least half its full
    private chunks (option dk_umma = 1, default), always with dk_umma = 2,
    never with 0 -- cfg2 shape (32 x 128 fp16, c = 64, 32 rows sharing 2048
    tokens), with a 1-token or a 512-token private tail per row."""
    import torch
    ca = ChunkAttention(32, 128, 64, 4096, 64, 8192, dtype=torch.float16, device=None)
    ca.set_option("dk_umma", umma)
    prompt = list(range(1, 2049))
    ids = [ca.add_sequence(prompt + [5000 + 7 * r + t for t in range(question + 1)])[0] for r in range(32)]
    ca.attend(ids)
    info = ca.schedule_info()
    assert info["dk"] == 1 and info["dk_um"] == expect
