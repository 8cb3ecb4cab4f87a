"""Row f4 on the device: the serving loop (iteration-based batching with
Poisson arrivals, requests joining and leaving) runs a few
dozen iterations; at every iteration the prefill-with-prefix-lookup outputs
(causal oracle C4) and the decode-step outputs (oracle C1) of sampled rows are
checked, and at the end the allocator drains."""
import numpy as np
import pytest
import torch

import synth
from oracle.attention import attend_heads_fp64, default_scale
from oracle.prefill import causal_prefill_fp64

pytestmark = pytest.mark.gpu


def test_serving_loop_outputs_and_drain():
    from paper_2402_15220_b200 import ChunkAttention
    from paper_2402_15220_b200.serving import ServingLoop, poisson_trace
    dev = torch.device("cuda", 0)
    h, d, c, seed = 4, 128, 64, 0
    n_p, n_s, n_c = 200, 128, 6
    ca = ChunkAttention(h, d, c, 400, 8, n_p + n_c + 2, dtype=torch.float16, out_dtype=torch.float16, device=dev)
    trace = poisson_trace(seed, 12, 2000.0, n_p, n_s, n_c)
    scale = default_scale(d)
    stats = {"decode_rows": 0, "prefill_rows": 0, "max_err": 0.0, "joins": 0}

    def kv(toks):
        t = torch.tensor(toks)
        pos = torch.arange(len(toks))
        return (synth.kv_values(seed, synth.TID_K, t, pos, 1, h, d)[:, 0].numpy(),
                synth.kv_values(seed, synth.TID_V, t, pos, 1, h, d)[:, 0].numpy())

    def observe(it):
        toks = it["tokens"]
        ids = it["decode_ids"]
        out = it["decode_out"].double().cpu().numpy()
        q = it["decode_q"].double().cpu().numpy()
        for r in sorted({0, len(ids) - 1}):
            K, V = kv(toks[ids[r]])
            ref = attend_heads_fp64(q[r], K, V, scale)
            stats["max_err"] = max(stats["max_err"], float(np.abs(out[r] - ref).max()))
            stats["decode_rows"] += 1
        if it["prefill_out"] is not None:
            pq = it["prefill_q"].double().cpu().numpy()
            po = it["prefill_out"].double().cpu().numpy()
            row = 0
            for sid, first in zip(it["prefill_ids"], it["prefill_first"]):
                prompt = toks[sid][:-1]  # the prompt (the decode token came after the prefill)
                K, V = kv(prompt)
                nq = len(prompt) - first
                ref = causal_prefill_fp64(pq[row:row + nq], K, V, first, scale)
                stats["max_err"] = max(stats["max_err"], float(np.abs(po[row:row + nq] - ref).max()))
                stats["prefill_rows"] += nq
                stats["joins"] += 1
                row += nq

    m = ServingLoop(ca, b_max=4, seed=seed).run(trace, "shared", observer=observe)
    assert m.requests == 12 and m.peak_batch <= 4 and m.iterations >= 12
    assert stats["joins"] == 12 and stats["decode_rows"] > 0 and stats["prefill_rows"] > 0
    assert stats["max_err"] <= 2e-3, stats
    assert m.prefill_tokens_matched > 0  # later joiners reuse the shared system prompt
    st = ca.memory_stats()
    assert st["used"] == 0 and st["free"] == st["created"]
