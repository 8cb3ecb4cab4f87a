"""GPU parity at the north_star configs' real shapes (BASELINE.json configs[2]
and configs[3]) plus the remaining boundary checks: every comparison against
the fp64 oracle (reading A11 tolerances), tables against the replay
oracle C3 (byte for byte), the uploaded tables against the host-built ones."""
import random

import numpy as np
import pytest
import torch

import synth
from oracle.tree_model import TreeModel
from tests.gpu_workload import Harness, build_shared, decode_tokens

pytestmark = pytest.mark.gpu


# ------------------------------------------------------- configs[2]: sweep ---
@pytest.mark.parametrize("opts", ["", "dk=0", "dk_umma=2"])
@pytest.mark.parametrize("b", [8, 32])
@pytest.mark.parametrize("n_s", [0, 2048, 4096])
def test_config3_sweep_point_all_rows(n_s, b, opts):
    """The shared-prompt sweep at n_p = 4096: n_s shared tokens + (4096 - n_s)
    private question tokens per row, then one fused decode step (append +
    attend; the two-call path for dk=0): every row and head against C1."""
    if opts == "dk=0" and b == 8 and n_s == 2048:
        pytest.skip("covered by the neighbouring points")
    if opts == "dk_umma=2" and n_s == 0:
        pytest.skip("no chunk-first unit: the tcgen05 variant is not taken")
    hs = Harness(32, 128, 64, "f16", "f16", seed=31 + n_s // 1024, alpha=8.0,
                 max_chunks=b * 66 + 80, max_batch=64, max_seq_len=4200, opts=opts)
    ids = build_shared(hs, n_s, [4096 - n_s] * b)
    hs.step = 1
    toks = decode_tokens(hs, ids)
    if opts.startswith("dk=0"):
        hs.append(ids, toks)
        hs.check(ids, 2e-3)
    else:
        hs.append_attend(ids, toks, 2e-3)


# ----------------------------------------- configs[3]: two-level tree, real ---
@pytest.mark.parametrize("umma", [1, 2])
def test_config4_two_level_tree_real_shape(umma):
    """BASELINE configs[3] at its real shape (chunk-first units on the
    auto-selected variant, and forced onto tcgen05: CTAs with several jobs --
    the system run and group runs): 32 heads x 128, chunk 64, a
    1024-token system prompt shared by all 64 rows, 4 groups x 16 rows sharing
    1024 tokens of examples, questions of 1..63 tokens, 512 fused decode steps
    with completion targets U[64, 512]: a finished sequence is removed (evict)
    and replaced at once (b stays 64).  Checkpoints {0, 63, 64, 255, 511}:
    every row against C1 and the tables byte-exact against the replay oracle
    C3 of the same op log; at the end the allocator drains to used = 0."""
    rng = random.Random(4)
    c, H, steps = 64, 32, 512
    hs = Harness(H, 128, c, "f16", "f16", seed=4, alpha=8.0, max_chunks=16 + 64 + 64 * 12 + 64,
                 max_batch=64, max_seq_len=4096, opts=f"dk_umma={umma}")
    tm = TreeModel(c, 16 + 64 + 64 * 12 + 64)
    sys_p = synth.token_ids(4, synth.TAG_SYS, 0, 1024).tolist()
    groups = [synth.token_ids(4, synth.TAG_GROUP, g, 1024).tolist() for g in range(4)]
    live, target, k = [], {}, 0

    def spawn(g=None):
        nonlocal k
        g = rng.randrange(4) if g is None else g
        q = synth.token_ids(4, synth.TAG_PRIV, k, rng.randint(1, 63)).tolist()
        k += 1
        toks = sys_p + groups[g] + q
        sid, _ = hs.add(toks)
        tm.add_sequence(toks)
        live.append(sid)
        target[sid] = rng.randint(64, 512)

    for g in range(4):
        for _ in range(16):
            spawn(g)
    checks = {0, 63, 64, 255, 511}
    for step in range(steps):
        hs.step = step + 1
        toks = decode_tokens(hs, live)
        rows = list(range(len(live))) if step in checks else None
        hs.append_attend(live, toks, 2e-3 if rows else None, rows=rows)
        tm.append(live, toks)
        if step in checks:
            assert hs.ca.export_context() == tm.export()
        for sid in list(live):
            target[sid] -= 1
            if target[sid] == 0:
                hs.remove(sid)
                tm.remove_sequence(sid)
                live.remove(sid)
                spawn()
    for sid in list(live):
        hs.remove(sid)
        tm.remove_sequence(sid)
    st = hs.ca.memory_stats()
    assert st["used"] == 0 and st["free"] == st["created"]
    assert (st["used"], st["free"], st["created"], st["hwm"], st["waste_slots"]) == tm.memory_stats()


# --------------------------------------------------- boundary and corner ---
def test_download_tables_equal_host_blob():
    """The lazy upload lands byte for byte: after structural
    changes (adds, a remove, a chunk-full append) the device tables equal the
    host-built blob."""
    hs = Harness(4, 128, 64, "f16", "f16", seed=41, alpha=8.0)
    ids = build_shared(hs, 640, [3, 70, 0, 129, 63])
    hs.check(ids, 2e-3)
    assert np.array_equal(hs.ca.download_tables(), hs.ca.host_tables())
    hs.remove(ids[2])
    ids = ids[:2] + ids[3:]
    hs.check(ids, 2e-3)
    assert np.array_equal(hs.ca.download_tables(), hs.ca.host_tables())
    hs.step = 1
    hs.append(ids, decode_tokens(hs, ids))  # row 4 (63 private tokens) grows a chunk
    hs.check(ids, 2e-3)
    dev, host = hs.ca.download_tables(), hs.ca.host_tables()
    # the append kernel advanced the device lengths (authoritative between
    # rebuilds); every other table is the host's
    n = len(ids)
    assert np.array_equal(dev[:n], host[:n] + 1) and np.array_equal(dev[n:], host[n:])


def test_merge_many_contributions_fused():
    """The fused persistent kernel's merge with more than 32 contributions per
    row (the per-column path of merge_pending): 48 shared chunks, one per
    chunk-first split."""
    hs = Harness(2, 64, 16, "f16", "f16", seed=43, alpha=8.0, opts="dk=0,cf_splits=1")
    ids = build_shared(hs, 48 * 16, [3, 20, 0, 9])
    hs.check(ids, 2e-3)
    assert hs.ca.counters()["slots"] >= 4 * 33


def test_general_magnitude_kv():
    """fp16 K/V of general magnitude (Gaussian x 4, exactly representable
    after rounding): decode parity through the fused step and attend-only."""
    tables = {}

    def kv_fn(which, toks, pos):  # a function of (token, position) only: sharing stays valid
        if which not in tables:
            g = torch.Generator().manual_seed(int(which) * 7919 + 17)
            tables[which] = (torch.randn((4096, 4, 128), generator=g, dtype=torch.float64) * 4.0).to(torch.float16)
        x = tables[which][(toks.cpu() * 31 + pos.cpu() * 7) % 4096][:, None]
        return x.double()
    hs = Harness(4, 128, 64, "f16", "f16", seed=44, alpha=1.0, kv_fn=kv_fn)
    ids = build_shared(hs, 256, [5, 70, 0, 130])
    hs.check(ids, 2e-3)
    for st in range(1, 3):
        hs.step = st
        hs.append_attend(ids, decode_tokens(hs, ids), 2e-3)


@pytest.mark.parametrize("c", [80, 112])
def test_chunk_sizes_without_mma_seq_first(c):
    """ADVICE: chunk sizes the MMA seq-first kernel does not take (80, 112)
    run the SIMT consumers without the fused schedule (no hang) -- parity."""
    hs = Harness(2, 64, c, "f16", "f16", seed=45, alpha=8.0)
    ids = build_shared(hs, 3 * c, [0, 5, c + 7])
    hs.check(ids, 2e-3)
    hs.step = 1
    hs.append_attend(ids, decode_tokens(hs, ids), 2e-3)
