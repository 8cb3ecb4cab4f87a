"""Zero-copy check: append/attend with pinned host (UVA) q, k, v, out pointers
must give the same output as device buffers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import DecodeWorkload

dev = torch.device("cuda", 0)
outs = []
for host in (False, True):
    wl = DecodeWorkload(dev, steps=80)
    wl.fill()
    s = torch.cuda.current_stream().cuda_stream
    hk = wl.kn.cpu().pin_memory() if host else wl.kn
    hv = wl.vn.cpu().pin_memory() if host else wl.vn
    hq = wl.q.cpu().pin_memory() if host else wl.q
    out = torch.empty(tuple(wl.out.shape), dtype=wl.out.dtype).pin_memory() if host else wl.out
    for st in range(70):
        wl.ca.append_raw(wl.ids, wl.tokens[st], hk[st].data_ptr(), hv[st].data_ptr(), s)
        wl.ca.attend_raw(0, wl.ids, hq[st].data_ptr(), out.data_ptr(), s)
    torch.cuda.synchronize()
    outs.append(out.cpu().clone())
print("host-pointer path bitwise equal:", torch.equal(outs[0], outs[1]), float((outs[0].float() - outs[1].float()).abs().max()))
