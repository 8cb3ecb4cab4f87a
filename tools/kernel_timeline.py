"""Per-CTA timelines of the seq-first / chunk-first kernels (debug option
"trace": %globaltimer stamps written into the last 2 MiB of the workspace).

    python tools/kernel_timeline.py --step 400 [--opt sf_ctas_per_sm=1 ...]

Prints, for one decode step of the bench workload, the kernel span, the
per-CTA active span, the load latency (data ready - issue) of each unit and
the consumer gap between consecutive units."""
from __future__ import annotations

import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import DecodeWorkload, flush_l2, time_steps  # noqa: E402

TRACE_STRIDE, TRACE_CTAS, TRACE_UNITS = 128, 2048, 41


def summarise(tr, name, ncta):
    t = tr[:ncta].astype(np.int64)
    t0 = t[:, 0][t[:, 0] > 0].min()
    ends = t[:, 2]
    print(f"== {name}: {ncta} CTAs, kernel span {(ends.max() - t0) / 1e3:.2f} us")
    starts = (t[:, 0] - t0) / 1e3
    print(f"   CTA start offset us: min {starts.min():.2f} med {np.median(starts):.2f} max {starts.max():.2f}")
    print(f"   CTA active us: med {np.median((ends - t[:, 0]) / 1e3):.2f} max {((ends - t[:, 0]) / 1e3).max():.2f}")
    lat, gap, first, comp, waitc = [], [], [], [], []
    for c in range(ncta):
        issue = t[c, 3::3][:TRACE_UNITS]
        ready = t[c, 4::3][:TRACE_UNITS]
        done = t[c, 5::3][:TRACE_UNITS]
        ok = (issue > 0) & (ready > 0) & (done > 0)
        if not ok.any():
            continue
        first.append((ready[0] - t[c, 0]) / 1e3)
        prev_done = None
        for u in np.nonzero(ok)[0]:
            lat.append((ready[u] - issue[u]) / 1e3)
            comp.append((done[u] - ready[u]) / 1e3)
            if prev_done is not None:
                waitc.append(max(0, ready[u] - prev_done) / 1e3)
                gap.append((ready[u] - ready[prev_u]) / 1e3)
            prev_done, prev_u = done[u], u
    q = lambda v: f"p10 {np.percentile(v, 10):.2f} med {np.median(v):.2f} p90 {np.percentile(v, 90):.2f} mean {np.mean(v):.2f}" if v else "-"
    print(f"   first data after entry us: {q(first)}")
    print(f"   load latency (ready - issue) us: {q(lat)}")
    print(f"   consume time (done - ready) us: {q(comp)}")
    print(f"   consumer idle before unit (ready - prev done) us: {q(waitc)}")
    print(f"   gap between consecutive traced ready us: {q(gap)}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--step", type=int, default=400)
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--kernel", default="sf", choices=["sf", "cf"])
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    wl = DecodeWorkload(dev, steps=args.step + 2)
    for o in args.opt:
        k, v = o.split("=")
        wl.ca.set_option(k, int(v))
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)
    wl.fill()
    ms = time_steps(wl, args.step, flush, stream)
    print(f"steps 0..{args.step - 1}: mean {np.mean(ms) * 1e3:.1f} us/step, last {ms[-1] * 1e3:.1f}")
    wl.ca.set_option("trace", 1 if args.kernel == "sf" else 2)
    ws = wl.ca.workspace
    tr_t = ws[ws.numel() - 8 * TRACE_CTAS * TRACE_STRIDE:].view(torch.int64)
    tr_t.zero_()
    with torch.cuda.stream(stream):
        flush_l2(flush)
        wl.step(args.step, stream.cuda_stream)
    stream.synchronize()
    tr = tr_t.view(TRACE_CTAS, TRACE_STRIDE).cpu().numpy()
    ncta = int((tr[:, 0] > 0).sum())
    summarise(tr, args.kernel, ncta)


if __name__ == "__main__":
    main()
