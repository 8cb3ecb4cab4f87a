"""Where does a decode step's event-bracketed time go beyond the kernel's own
span?  Times the bench's fused step (append_attend) (a) after an L2 flush
(the bench's protocol), (b) back to back with no flush, (c) after a tiny
kernel that uses no shared memory, (d) after a flush plus a shared-memory-heavy
torch op, and reports the ncu-free device time of each."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from bench import DecodeWorkload, flush_l2

dev = torch.device("cuda", 0)
wl = DecodeWorkload(dev, steps=400)
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
small = torch.empty(1024, device=dev)
a = torch.randn(2048, 2048, device=dev, dtype=torch.float16)
stream = torch.cuda.Stream(dev)
sp = stream.cuda_stream


def run(label, pre, n=40, s0=0):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    with torch.cuda.stream(stream):
        for i in range(n):
            pre()
            evs[i][0].record(stream)
            wl.step(s0 + i, sp)
            evs[i][1].record(stream)
    stream.synchronize()
    ms = np.array([x.elapsed_time(y) for x, y in evs]) * 1e3
    print(f"{label:40s} mean {ms.mean():6.1f} us  med {np.median(ms):6.1f}  min {ms.min():6.1f}")


wl.fill()
run("warm", lambda: flush_l2(flush), 20, 0)
for opt in ([], [("dk", 0)]):
    for k, v in opt:
        wl.ca.set_option(k, v)
    wl.one_launch = not opt
    tag = "K5" if not opt else "persistent(dk=0)"
    wl.fill()
    run(f"{tag}: flush (bench protocol)", lambda: flush_l2(flush), 40, 0)
    wl.fill()
    run(f"{tag}: back to back, no flush", lambda: None, 40, 0)
    wl.fill()
    run(f"{tag}: after a tiny kernel", lambda: small.add_(1.0), 40, 0)
    wl.fill()
    run(f"{tag}: flush + fp16 GEMM (smem-heavy)", lambda: (flush_l2(flush), torch.mm(a, a)), 40, 0)
