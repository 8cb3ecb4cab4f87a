"""What does the append cost inside a decode step?  Per-step GPU time of full
steps (append + attend, PDL chain) around step S vs attend-only and
append-only launches on the cache state of step S (same flush between steps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from bench import DecodeWorkload, flush_l2, time_steps

S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
opts = [o.split("=") for o in sys.argv[2:]]
dev = torch.device("cuda", 0)
wl = DecodeWorkload(dev, steps=S + 40)
for k, v in opts:
    wl.ca.set_option(k, int(v))
flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size // 4, dtype=torch.float32, device=dev)
stream = torch.cuda.Stream(dev)
wl.fill()
ms = time_steps(wl, S + 20, flush, stream)
full = np.mean(ms[S - 8:S + 8]) * 1e3
sp = stream.cuda_stream


def timed(fn, n=40):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    with torch.cuda.stream(stream):
        for i in range(n):
            flush_l2(flush)
            evs[i][0].record(stream)
            fn(i)
            evs[i][1].record(stream)
    stream.synchronize()
    return np.mean([a.elapsed_time(b) for a, b in evs]) * 1e3


att = timed(lambda i: wl.ca.attend_raw(0, wl.ids, wl.q[S].data_ptr(), wl.out.data_ptr(), sp))
print(f"step ~{S}: full step {full:.1f} us | attend only (state of step {S + 20}) {att:.1f} us", flush=True)
