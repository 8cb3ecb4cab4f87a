"""Multi-rank host logic on CPU (gloo, world size 2): head slicing, the output
gather + permutation (checked against the fp64 oracle computed per rank on its
heads), and identical prefix trees on every rank without collectives."""
import os
import random
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.attention import attend_heads_fp64, default_scale
        from paper_2402_15220_b200.dist import ShardedChunkAttention, gather_heads, head_range

        H, d, c, seed = 8, 64, 4, 3
        sh = ShardedChunkAttention(H, d, c, max_chunks=500, max_batch=64, max_seq_len=512, device=None)
        assert (sh.h0, sh.h1) == head_range(H, world, rank)
        # identical op stream on every rank (host-only handles: tree + tables)
        rng = random.Random(7)
        prompt = [rng.randint(1, 999) for _ in range(3 * c)]
        seqs = {}
        for i in range(6):
            toks = prompt[:rng.randint(0, len(prompt))] + [rng.randint(1, 999) for _ in range(rng.randint(1, 9))]
            sid, _ = sh.add_sequence(toks)
            seqs[sid] = toks
        for step in range(7):
            ids = sorted(seqs)
            new = [rng.randint(1, 999) for _ in ids]
            sh.append_kv(ids, new)
            for s, t in zip(ids, new):
                seqs[s].append(t)
            if step == 3:
                victim = ids[2]
                sh.remove_sequence(victim)
                del seqs[victim]
        ok = sh.tables_consistent()
        # gather + permutation: each rank computes the oracle for ITS heads only
        ids = sorted(seqs)
        q = synth.q_values(seed, torch.tensor(ids), 0, 1, H, d, alpha=8.0)[:, 0]
        out_local = np.zeros((len(ids), sh.h1 - sh.h0, d))
        full_ref = np.zeros((len(ids), H, d))
        for r, s in enumerate(ids):
            toks = torch.tensor(seqs[s])
            pos = torch.arange(len(toks))
            K = synth.kv_values(seed, synth.TID_K, toks, pos, 1, H, d)[:, 0].numpy()
            V = synth.kv_values(seed, synth.TID_V, toks, pos, 1, H, d)[:, 0].numpy()
            full_ref[r] = attend_heads_fp64(q[r].numpy(), K, V, default_scale(d))
            Kl = synth.kv_values(seed, synth.TID_K, toks, pos, 1, sh.h1 - sh.h0, d, head_offset=sh.h0)[:, 0].numpy()
            Vl = synth.kv_values(seed, synth.TID_V, toks, pos, 1, sh.h1 - sh.h0, d, head_offset=sh.h0)[:, 0].numpy()
            out_local[r] = attend_heads_fp64(q[r, sh.h0:sh.h1].numpy(), Kl, Vl, default_scale(d))
        gathered = gather_heads(torch.from_numpy(out_local)).numpy()
        results[rank] = (ok, float(np.abs(gathered - full_ref).max()), sh.ca.export_context())
    finally:
        dist.destroy_process_group()


def test_two_rank_head_sharding_gloo():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert len(results) == world
    for r in range(world):
        ok, err, text = results[r]
        assert ok, "ranks built different prefix trees"
        assert err < 1e-12, err
    assert results[0][2] == results[1][2]


def test_head_range_validation():
    from paper_2402_15220_b200.dist import head_range
    assert head_range(32, 8, 3) == (12, 16)
    with pytest.raises(ValueError):
        head_range(32, 3, 0)
