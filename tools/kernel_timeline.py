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

TRACE_STRIDE, TRACE_CTAS, TRACE_UNITS = 128, 2048, 31
CF_TILE_BYTES = 2 * 64 * 128 * 2  # cfg2 chunk-first unit: K + V tile of one (chunk, head)


def summarise(tr, name, ncta):
    t = tr[:ncta].astype(np.int64)
    t0 = t[:, 0][t[:, 0] > 0].min()
    ends = t[:, 2]
    print(f"== {name}: {ncta} CTAs, kernel span {(ends.max() - t0) / 1e3:.2f} us")
    starts = (t[:, 0] - t0) / 1e3
    print(f"   CTA start offset us: min {starts.min():.2f} med {np.median(starts):.2f} max {starts.max():.2f}")
    print(f"   CTA active us: med {np.median((ends - t[:, 0]) / 1e3):.2f} max {((ends - t[:, 0]) / 1e3).max():.2f}")
    eo = (ends - t0) / 1e3
    print(f"   CTA end offset us: p10 {np.percentile(eo, 10):.2f} med {np.median(eo):.2f} "
          f"p90 {np.percentile(eo, 90):.2f} max {eo.max():.2f}")
    tails = []
    for c in range(ncta):
        d = t[c, 5::4][:TRACE_UNITS]
        d = d[d > 0]
        if d.size:
            tails.append((ends[c] - d.max()) / 1e3)
    if tails:
        print(f"   tail after last traced unit us (finalize/fixup): med {np.median(tails):.2f} "
              f"p90 {np.percentile(tails, 90):.2f} max {max(tails):.2f}")
    lat, gap, first, comp, waitc = [], [], [], [], []
    for c in range(ncta):
        issue = t[c, 3::4][:TRACE_UNITS]
        ready = t[c, 4::4][:TRACE_UNITS]
        done = t[c, 5::4][:TRACE_UNITS]
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
    fi = [(t[c, 3] - t[c, 0]) / 1e3 for c in range(ncta) if t[c, 3] > 0]
    print(f"   first issue after entry us: {q(fi)}")
    print(f"   first data after entry us: {q(first)}")
    print(f"   load latency (ready - issue) us: {q(lat)}")
    print(f"   consume time (done - ready) us: {q(comp)}")
    print(f"   consumer idle before unit (ready - prev done) us: {q(waitc)}")
    print(f"   gap between consecutive traced ready us: {q(gap)}")
    # phases per CTA: chunk-first units (64 KiB K+V tiles first in the CTA's
    # list), seq-first units, the merge phase (tr[127] = after settle, tr[2] = end)
    cf_end, sf_end, mg_start, mg_len, n_cf = [], [], [], [], []
    for c in range(ncta):
        by_c = t[c, 6::4][:TRACE_UNITS]
        done = t[c, 5::4][:TRACE_UNITS]
        k = 0
        while k < len(by_c) and by_c[k] == CF_TILE_BYTES and done[k] > 0:
            k += 1
        n_cf.append(k)
        if k:
            cf_end.append((done[k - 1] - t0) / 1e3)
        dd = done[done > 0]
        if dd.size > k:
            sf_end.append((dd.max() - t0) / 1e3)
        if t[c, TRACE_STRIDE - 1] > 0:
            mg_start.append((t[c, TRACE_STRIDE - 1] - t0) / 1e3)
            mg_len.append((ends[c] - t[c, TRACE_STRIDE - 1]) / 1e3)
    q2 = lambda v: f"med {np.median(v):.2f} p90 {np.percentile(v, 90):.2f} max {max(v):.2f}" if v else "-"
    print(f"   chunk-first units per CTA: {q2(n_cf)}; CTAs with any: {sum(1 for x in n_cf if x)}")
    print(f"   chunk-first phase end us: {q2(cf_end)}")
    print(f"   seq-first phase end us: {q2(sf_end)}")
    print(f"   merge phase start us: {q2(mg_start)}; merge phase length us: {q2(mg_len)}")
    # aggregate data arrival rate over the kernel (bytes of each unit at its ready time)
    rd = t[:, 4:4 + 4 * TRACE_UNITS:4].ravel()
    by = t[:, 6:6 + 4 * TRACE_UNITS:4].ravel()
    ok = (rd > 0) & (by > 0)
    if ok.any():
        rel = (rd[ok] - t0) / 1e3
        span = (ends.max() - t0) / 1e3
        bins = np.arange(0, span + 2, 2.0)
        hist, _ = np.histogram(rel, bins=bins, weights=by[ok].astype(np.float64))
        print(f"   traced bytes {by[ok].sum() / 1e6:.1f} MB; arrival TB/s per 2 us bin:")
        print("   " + " ".join(f"{h / 2e-6 / 1e12:.1f}" for h in hist))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--step", type=int, default=400)
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--kernel", default="sf", choices=["sf", "cf"])
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--n-shared", dest="n_shared", type=int, default=2048)
    ap.add_argument("--question", type=int, default=0)
    ap.add_argument("--flush", default="write", choices=["write", "clean"],
                    help="clean: write then read the flush buffer (no dirty lines left in L2)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    wl = DecodeWorkload(dev, steps=args.step + 2, b=args.batch, n_shared=args.n_shared, question=args.question)
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
        if args.flush == "clean":
            flush.sum()
        wl.step(args.step, stream.cuda_stream)
    stream.synchronize()
    tr = tr_t.view(TRACE_CTAS, TRACE_STRIDE).cpu().numpy()
    ncta = int((tr[:, 0] > 0).sum())
    info = wl.ca.schedule_info()
    print("schedule:", info)
    summarise(tr, args.kernel, ncta)
    if info["dk"]:  # K5: per cluster rank (blockIdx = group * cs + rank)
        cs = info["dk_cs"]
        t = tr[:ncta].astype(np.int64)
        t0 = t[:, 0][t[:, 0] > 0].min()
        for r in range(cs):
            sel = t[r::cs]
            nun = [(x[5::4][:TRACE_UNITS] > 0).sum() for x in sel]
            cdone = (sel[:, 1] - t0) / 1e3
            mstart = (sel[:, TRACE_STRIDE - 1] - t0) / 1e3
            end = (sel[:, 2] - t0) / 1e3
            mloop = (sel[:, TRACE_STRIDE - 2] - t0) / 1e3
            mload = (sel[:, TRACE_STRIDE - 8] - t0) / 1e3
            alld = (sel[:, TRACE_STRIDE - 3] - t0) / 1e3
            cwait = (sel[:, TRACE_STRIDE - 4] - t0) / 1e3
            pushd = (sel[:, TRACE_STRIDE - 5] - t0) / 1e3
            x = sel[0]
            seq = []
            for u in range(TRACE_UNITS):
                if x[3 + 4 * u] == 0 and x[4 + 4 * u] == 0:
                    break
                seq.append(f"[{(x[3 + 4 * u] - t0) / 1e3:.1f}/{(x[4 + 4 * u] - t0) / 1e3:.1f}/"
                           f"{(x[5 + 4 * u] - t0) / 1e3:.1f} {x[6 + 4 * u] // 1024}K]")
            print(f"   rank {r} CTA 0 units issue/ready/done: " + " ".join(seq))
            ex = {"firstQ": TRACE_STRIDE - 6, "cf_epi": TRACE_STRIDE - 7, "firstS": TRACE_STRIDE - 10,
                  "mergesync": TRACE_STRIDE - 9}
            print("   rank %d (tcgen05 marks, median): " % r + " ".join(
                f"{k} {np.median((sel[:, w] - t0) / 1e3):.2f}" for k, w in ex.items() if (sel[:, w] > 0).any()))
            print(f"   rank {r}: traced units med {np.median(nun):.0f}; consumers done med {np.median(cdone):.2f} "
                  f"max {cdone.max():.2f}; all consumers {np.median(alld):.2f}; cluster wait {np.median(cwait):.2f}; "
                  f"pushed {np.median(pushd):.2f}; merge start med {np.median(mstart):.2f}; first loads med {np.median(mload):.2f}; "
                  f"loop done med {np.median(mloop):.2f}; "
                  f"end med {np.median(end):.2f} "
                  f"max {end.max():.2f} us")


if __name__ == "__main__":
    main()
