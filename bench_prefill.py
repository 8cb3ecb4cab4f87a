#!/usr/bin/env python
"""Prefill attention with prefix lookup on one
B200: b sequences whose prompts share an n_s-token system prompt, each with a
private q_len-token suffix (Llama-2-7B attention shape: 32 heads x 128, fp16,
chunk 64).  Synthetic, seeded inputs (DESIGN.md input recipe).

  lookup     prefix matching on: the first sequence prefills its whole prompt,
             the others only their suffix queries (the shared chunks' K/V are
             matched, never recomputed; their queries skip attention)
  no_lookup  prefix matching off (the non-shared paged layout): every sequence
             prefills its whole prompt

Timed: one chunkattn_prefill_attend over the whole batch (one launch), CUDA
events on the launch stream, L2 flushed between iterations.  Reported per
mode: query tokens/s, attention TFLOP/s (4 d (p + 1) per query and head: QK^T
and PV, 2 flop per FMA) against the tensor roofline (MEASURED_PEAKS.json bf16
burst; fp16 has the same nominal rate), and the speedup of lookup.

    python bench_prefill.py [--batch 32] [--n-shared 2048] [--q-len 128]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

_CLOCKS = None

import synth  # noqa: E402
from bench import flush_l2  # noqa: E402


def run(mode, b, n_s, q_len, h=32, d=128, c=64, iters=20, seed=0):
    from paper_2402_15220_b200 import ChunkAttention
    dev = torch.device("cuda", 0)
    n = n_s + q_len
    per_seq = (n + c - 1) // c
    ca = ChunkAttention(h, d, c, per_seq * b + 8, b, n + 1, dtype=torch.float16, out_dtype=torch.float16,
                        prefix_match=(mode == "lookup"), device=dev)
    prompt = synth.token_ids(seed, synth.TAG_SYS, 0, n_s, device=dev)
    ids, firsts, pos_list = [], [], []
    for r in range(b):
        toks = torch.cat([prompt, synth.token_ids(seed, synth.TAG_PRIV, r, q_len, device=dev)])
        tl = toks.tolist()
        m = ca.match_prefix(tl)
        pos = torch.arange(m, n, device=dev)
        k = synth.kv_values(seed, synth.TID_K, toks[m:], pos, 1, h, d, device=dev).to(torch.float16)
        v = synth.kv_values(seed, synth.TID_V, toks[m:], pos, 1, h, d, device=dev).to(torch.float16)
        sid, matched = ca.add_sequence(tl, k.contiguous(), v.contiguous(), kv_first_pos=m)
        ids.append(sid)
        firsts.append(matched)
        pos_list.append(torch.arange(matched, n))
    positions = torch.cat(pos_list)
    nq = int(positions.numel())
    g = torch.Generator(device=dev).manual_seed(seed + 1)
    q = torch.randn((nq, h, d), generator=g, device=dev, dtype=torch.float32).to(torch.float16)
    out = torch.empty_like(q)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        for _ in range(3):
            ca.prefill_attend(ids, firsts, q, out=out)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        for a, e in evs:
            flush_l2(flush)
            a.record(stream)
            ca.prefill_attend(ids, firsts, q, out=out)
            e.record(stream)
    stream.synchronize()
    us = statistics.median([a.elapsed_time(e) * 1e3 for a, e in evs])
    flops = 4.0 * d * h * float((positions + 1).sum())
    peak = 1672.4
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            peak = json.load(f).get("bf16_tflops", peak)
    tf = flops / (us * 1e-6) / 1e12
    return {"mode": mode, "b": b, "n_shared": n_s, "q_len": q_len, "h": h, "d": d, "c": c, "dtype": "f16",
            "queries": nq, "matched_tokens": int(sum(firsts)), "us_median": us, "query_tokens_per_s": nq / (us * 1e-6),
            "prompt_tokens_per_s": b * n / (us * 1e-6), "tflops": tf,
            "roofline": {"bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops (fp16 same nominal rate)"}}


def main():
    global _CLOCKS
    from bench import ClockSampler
    _CLOCKS = ClockSampler(0)
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--n-shared", dest="n_shared", type=int, default=2048)
    ap.add_argument("--q-len", dest="q_len", type=int, default=128)
    args = ap.parse_args()
    rows = [run(m, args.batch, args.n_shared, args.q_len) for m in ("lookup", "no_lookup")]
    rows[0]["speedup_vs_no_lookup"] = rows[1]["us_median"] / rows[0]["us_median"]
    for r in rows:
        r["clocks"] = _CLOCKS.snapshot()
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
