#!/usr/bin/env python
"""Serving-loop workload (tab:e2e_latency
shape) on one B200: Poisson arrivals, iteration-based batching with at most
b_max = 32 running requests, prompts of n_p tokens whose first n_s are a shared
system prompt, n_c completion tokens each; Llama-2-7B attention shape (32 x
128, fp16, chunk 64), synthetic seeded K/V/Q, attention work only (no model
weights: the clock is the device time of each iteration's prefill-with-lookup
and decode attention).  Both modes replay the identical request trace:

  shared      prefix matching on (PAKV + TPP, the default library)
  monolithic  prefix matching off (every request owns its KV: the paper's
              non-shared baseline)

Prints one JSON line per (n_s, mode) with normalised latency (ms of attention
per completion token, including queueing), peak KV bytes / chunks / batch, and
the shared-vs-monolithic ratios (KV memory -70..90%).

    python bench_serve.py [--requests 64] [--rps 2000] [--n-p 2048] [--n-c 256]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

_CLOCKS = None


def run_mode(trace, prefix_match, b_max, n_p, n_c, h=32, d=128, c=64):
    from paper_2402_15220_b200 import ChunkAttention
    from paper_2402_15220_b200.serving import ServingLoop
    dev = torch.device("cuda", 0)
    per_seq = (n_p + n_c + c - 1) // c + 1
    ca = ChunkAttention(h, d, c, per_seq * (b_max + 2) + 64, b_max + 2, n_p + n_c + 1, dtype=torch.float16,
                        out_dtype=torch.float16, prefix_match=prefix_match, device=dev)
    m = ServingLoop(ca, b_max).run(trace, "shared" if prefix_match else "monolithic")
    ca.close()
    del ca
    torch.cuda.empty_cache()
    return m


def main():
    global _CLOCKS
    from bench import ClockSampler
    _CLOCKS = ClockSampler(0)
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=64)
    ap.add_argument("--rps", type=float, default=2000.0, help="Poisson arrival rate (requests / s of attention time)")
    ap.add_argument("--n-p", dest="n_p", type=int, default=2048)
    ap.add_argument("--n-s", dest="n_s", type=int, action="append", default=None)
    ap.add_argument("--n-c", dest="n_c", type=int, default=256)
    ap.add_argument("--b-max", dest="b_max", type=int, default=32)
    args = ap.parse_args()
    from paper_2402_15220_b200.serving import poisson_trace
    for n_s in args.n_s or [0, 1024, 2048]:
        trace = poisson_trace(0, args.requests, args.rps, args.n_p, n_s, args.n_c)
        res = {}
        for pm in (True, False):
            m = run_mode(trace, pm, args.b_max, args.n_p, args.n_c)
            res[m.mode] = m
        for mode, m in res.items():
            line = {"workload": "serve_poisson", "mode": mode, "n_p": args.n_p, "n_s": n_s, "n_c": args.n_c,
                    "requests": m.requests, "rps": args.rps, "b_max": args.b_max, "h": 32, "d": 128, "c": 64,
                    "dtype": "f16", "data": "synthetic",
                    "normalized_latency_ms_per_tok": m.normalized_latency_ms_per_tok,
                    "mean_latency_ms": m.mean_latency_ms, "makespan_ms": m.makespan_ms,
                    "completion_tokens_per_s": m.completion_tokens / (m.makespan_ms * 1e-3),
                    "peak_batch": m.peak_batch, "peak_kv_chunks": m.peak_kv_chunks, "peak_kv_bytes": m.peak_kv_bytes,
                    "prefill_tokens_computed": m.prefill_tokens_computed,
                    "prefill_tokens_matched": m.prefill_tokens_matched, "iterations": m.iterations,
                    "clock": "device time of each iteration's attention launches (CUDA events); no model weights"}
            if mode == "shared":
                mono = res["monolithic"]
                line["kv_bytes_ratio_vs_monolithic"] = m.peak_kv_bytes / max(1, mono.peak_kv_bytes)
                line["latency_ratio_vs_monolithic"] = m.normalized_latency_ms_per_tok / max(
                    1e-12, mono.normalized_latency_ms_per_tok)
            line["clocks"] = _CLOCKS.snapshot()
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
