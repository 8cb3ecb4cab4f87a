#!/usr/bin/env python
"""Kernel-latency sweep vs shared-prompt length (BASELINE.json configs[2],
configs[4]; PAPER.md tab:kernel_latency layout).

For each point: b sequences of n_p prompt tokens whose first n_s are shared,
one decode token appended, then the two-phase attention timed alone (CUDA
events, L2 flushed before every timed call) for three modes of the same
library:
  chunk  ChunkAttention (PAKV + TPP)
  b0     prefix matching off: every sequence owns private copies -- the
         non-shared paged layout (the paper's PagedAttn)
  b1     physically shared chunks, no chunk-first phase (share_threshold = inf;
         the paper's PagedAttn*)
Prints one JSON line per point and a markdown table (profiles/ keeps a copy).

    python bench_sweep.py [--quick] [--points tab|cfg3|cfg5|all]
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

from bench import DecodeWorkload, flush_l2, load_peaks  # noqa: E402


def time_attend(wl: DecodeWorkload, iters: int, flush, stream) -> list[float]:
    sp = stream.cuda_stream
    q = wl.q[0]
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    with torch.cuda.stream(stream):
        for i in range(iters):
            flush_l2(flush)
            evs[i][0].record(stream)
            wl.ca.attend_raw(0, wl.ids, q.data_ptr(), wl.out.data_ptr(), sp)
            evs[i][1].record(stream)
    stream.synchronize()
    return [a.elapsed_time(b) * 1e3 for a, b in evs]  # us


def run_point(dev, b, n_p, n_s, mode, iters, flush, stream, c=64, opts=()):
    wl = DecodeWorkload(dev, b=b, n_shared=n_s, question=n_p - n_s, steps=2, mode=mode)
    for o in opts:
        key, val = o.split("=")
        wl.ca.set_option(key, int(val))
    wl.fill()
    with torch.cuda.stream(stream):
        wl.step(0, stream.cuda_stream)  # one decode token: context n_p + 1, attention after the append
    stream.synchronize()
    time_attend(wl, 3, flush, stream)  # warm-up
    us = time_attend(wl, iters, flush, stream)
    shape = wl.shape_at(0)
    bytes_alg = shape.unique_bytes()
    med = statistics.median(us)
    stats = wl.ca.memory_stats()
    del wl
    torch.cuda.empty_cache()
    return {"b": b, "n_p": n_p, "n_s": n_s, "mode": mode, "us_median": med, "us_p10": sorted(us)[len(us) // 10],
            "us_p90": sorted(us)[(9 * len(us)) // 10], "bytes_alg": bytes_alg,
            "gbs_alg": bytes_alg / (med * 1e-6) / 1e9, "tokens_per_s": b / (med * 1e-6),
            "kv_chunks_used": stats["used"], "kv_bytes": stats["kv_bytes"]}


def main():
    global _CLOCKS
    from bench import ClockSampler
    _CLOCKS = ClockSampler(0)
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", default="all", choices=["tab", "cfg3", "cfg5", "all"])
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--out", default=None)
    ap.add_argument("--opt", action="append", default=[], help="library option key=value (ChunkAttn mode only)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)
    peak, src, _ = load_peaks()
    pts = []
    if args.points in ("tab", "all"):  # tab:kernel_latency grid, b = 32
        for n_p in (1024, 2048, 4096):
            for n_s in (0, n_p // 2, 3 * n_p // 4, n_p):
                pts.append((32, n_p, n_s))
    if args.points in ("cfg3", "all"):  # configs[2]: n_s sweep x batch 8 / 16 at n_p = 4096
        for b in (8, 16):
            for n_s in (0, 1024, 2048, 4096):
                pts.append((b, 4096, n_s))
    if args.points in ("cfg5", "all"):  # configs[4] on one GPU: b = 256, n_s = 4096, 64-token question
        pts.append((256, 4096 + 64, 4096))
    rows = []
    for (b, n_p, n_s) in pts:
        res = {}
        for mode in ("chunk", "b1", "b0"):
            r = run_point(dev, b, n_p, n_s, mode, args.iters, flush, stream,
                          opts=args.opt if mode == "chunk" else ())
            res[mode] = r
        for mode, r in res.items():
            r["speedup_vs_b0"] = res["b0"]["us_median"] / r["us_median"]
            r["frac_hbm"] = r["gbs_alg"] / peak
            r["clocks"] = _CLOCKS.snapshot()
            print(json.dumps(r), flush=True)
            rows.append(r)
    lines = ["| b | n_p | n_s | ChunkAttn µs | B1 (shared, no TPP) µs | B0 (non-shared paged) µs | speedup vs B0 | "
             "ChunkAttn GB/s (alg) | frac of HBM |", "|---|---|---|---|---|---|---|---|---|"]
    for i in range(0, len(rows), 3):
        ch, b1, b0 = rows[i], rows[i + 1], rows[i + 2]
        lines.append(f"| {ch['b']} | {ch['n_p']} | {ch['n_s']} | {ch['us_median']:.1f} | {b1['us_median']:.1f} | "
                     f"{b0['us_median']:.1f} | {ch['speedup_vs_b0']:.2f}x | {ch['gbs_alg']:.0f} | "
                     f"{ch['frac_hbm']:.2f} |")
    table = "\n".join(lines)
    print(table)
    if args.out:
        with open(args.out, "w") as f:
            f.write(f"# Kernel latency sweep (attention only, L2 flushed, median of {args.iters}; peak {peak} GB/s "
                    f"{src})\n\n{table}\n")


if __name__ == "__main__":
    main()
