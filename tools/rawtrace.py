"""Raw per-CTA trace words of one K5 step (option "trace"): the tcgen05
variant's chunk-first pipeline marks and the merge-phase marks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import DecodeWorkload, flush_l2, time_steps
step = int(sys.argv[1]) if len(sys.argv) > 1 else 10
opts = sys.argv[2:]
dev = torch.device("cuda", 0)
wkw = {o.split("=")[0][3:]: int(o.split("=")[1]) for o in opts if o.startswith("wl_")}  # wl_d=64 wl_h=64: workload shape
wl = DecodeWorkload(dev, steps=step + 4, **wkw)
for o in opts:
    if o.startswith("wl_"):
        continue
    k, v = o.split("=")
    wl.ca.set_option(k, int(v))
flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size // 4, dtype=torch.float32, device=dev)
stream = torch.cuda.Stream(dev)
wl.fill()
time_steps(wl, step, flush, stream)
wl.ca.set_option("trace", 1)
ws = wl.ca.workspace
tr_t = ws[ws.numel() - 8 * 2048 * 128:].view(torch.int64)
tr_t.zero_()
with torch.cuda.stream(stream):
    flush_l2(flush); flush.sum()
    wl.step(step, stream.cuda_stream)
stream.synchronize()
tr = tr_t.view(2048, 128).cpu().numpy().astype(np.int64)
n = int((tr[:, 0] > 0).sum())
t0 = tr[:n, 0][tr[:n, 0] > 0].min()
rel = lambda x: np.where(x > 0, (x - t0) / 1e3, np.nan)
marks = dict(entry=0, cons_done=1, end=2, firstQ=122, cf_epi=121, firstS=118, mergesync=119, allcons=125, clw=124,
             pushed=123, mstart=127, firstld=120, loopdone=126, s3_issue0=116, s3_issue1=117)
print("CTA0 npre + 100 nk + 10000 nv:", tr[0, 115], " CTA1:", tr[1, 115])
print("median over CTAs:", {k: round(float(np.nanmedian(rel(tr[:n, w]))), 2) for k, w in marks.items()})
print("max over CTAs:", {k: round(float(np.nanmax(rel(tr[:n, w]))), 2) for k, w in marks.items()})
print("chunk-first unit k: K issued / V issued / K in smem (issuer) / S ready / P done / P seen by issuer  (CTA 0 | medians)")
for k in range(14):
    if tr[0, 3 + 4 * k] == 0:
        break
    cols = [3 + 4 * k, 102 + k, 70 + k, 4 + 4 * k, 5 + 4 * k, 86 + k]
    print(k, " ".join(f"{rel(tr[0, c]):6.2f}" for c in cols), " | ", " ".join(f"{np.nanmedian(rel(tr[:n, c])):6.2f}" for c in cols))
