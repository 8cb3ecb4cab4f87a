"""Two ranks on the GPU (torch.multiprocessing, gloo for the collectives so
both ranks can share the one GPU of the test box): the head split
(ShardedChunkAttention: every rank replays the op stream, holds its heads,
one all-gather per step; byte-identical tables checked by a hash all-gather)
and the row split of one batch (RowShardedChunkAttention), each against the
fp64 oracle on all heads and rows after fused decode steps."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _seqs(seed, c):
    """Two prompt groups (2 and 3 full chunks), private questions of 0..c+5."""
    p0 = synth.token_ids(seed, synth.TAG_SYS, 0, 2 * c).tolist()
    p1 = synth.token_ids(seed, synth.TAG_SYS, 1, 3 * c).tolist()
    out = []
    for i, q in enumerate([0, 5, c + 5, 3, 17, c, 1]):
        pre = p0 if i % 2 == 0 else p1
        out.append(pre + synth.token_ids(seed, synth.TAG_PRIV, i, q).tolist())
    return out


def _oracle(seed, toks_of, ids, q, H, d):
    from oracle.attention import attend_heads_fp64, default_scale
    ref = np.zeros((len(ids), H, d))
    for r, s in enumerate(ids):
        t = torch.tensor(toks_of[s])
        pos = torch.arange(len(t))
        K = synth.kv_values(seed, synth.TID_K, t, pos, 1, H, d)[:, 0].numpy()
        V = synth.kv_values(seed, synth.TID_V, t, pos, 1, H, d)[:, 0].numpy()
        ref[r] = attend_heads_fp64(q[r].numpy(), K, V, default_scale(d))
    return ref


def _worker(rank, world, port, kind, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2402_15220_b200.dist import RowShardedChunkAttention, ShardedChunkAttention
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        H, d, c, seed = 8, 128, 64, 5
        cls = ShardedChunkAttention if kind == "heads" else RowShardedChunkAttention
        sh = cls(H, d, c, max_chunks=300, max_batch=16, max_seq_len=1024, device=dev)
        toks_of = {}
        for toks in _seqs(seed, c):
            t = torch.tensor(toks)
            pos = torch.arange(len(t))
            k = synth.kv_values(seed, synth.TID_K, t, pos, 1, H, d).to(dev, torch.float16)
            v = synth.kv_values(seed, synth.TID_V, t, pos, 1, H, d).to(dev, torch.float16)
            sid = sh.add_sequence(toks, k, v)
            sid = sid[0] if isinstance(sid, tuple) else sid
            toks_of[sid] = list(toks)
        errs = []
        ids = sorted(toks_of)
        for step in range(1, 4):
            ids = ids[::-1] if step == 2 else ids
            new = [int(synth.hash_py(seed, synth.TAG_DECODE, s, step) % 31999 + 1) for s in ids]
            pos = torch.tensor([len(toks_of[s]) for s in ids])
            kn = synth.kv_values(seed, synth.TID_K, torch.tensor(new), pos, 1, H, d)[:, 0].to(dev, torch.float16)
            vn = synth.kv_values(seed, synth.TID_V, torch.tensor(new), pos, 1, H, d)[:, 0].to(dev, torch.float16)
            for s, t in zip(ids, new):
                toks_of[s].append(t)
            q = synth.q_values(seed, torch.tensor(ids), step, 1, H, d, alpha=8.0)[:, 0]
            out = sh.append_attend(ids, new, kn.contiguous(), vn.contiguous(), q.to(dev, torch.float16).contiguous())
            torch.cuda.synchronize()
            errs.append(float(np.abs(out.double().cpu().numpy() - _oracle(seed, toks_of, ids, q, H, d)).max()))
        same = sh.tables_consistent() if kind == "heads" else True
        results[rank] = (max(errs), same)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["heads", "rows"])
def test_two_ranks_on_gpu(kind):
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), kind, results), nprocs=world, join=True)
    assert len(results) == world
    for r in range(world):
        err, same = results[r]
        assert same, "ranks built different prefix trees"
        assert err <= 2e-3, (r, err)
