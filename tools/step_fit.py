"""Per-step GPU time of the bench's pass A vs the step's algorithmic bytes:
least-squares fit t = t0 + bytes / BW (fixed floor t0 and streaming rate BW)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from bench import DecodeWorkload, time_steps

K = int(sys.argv[1]) if len(sys.argv) > 1 else 512
opts = [a.split("=") for a in sys.argv[2:]]
dev = torch.device("cuda", 0)
wl = DecodeWorkload(dev, steps=K)
for k, v in opts:
    wl.ca.set_option(k, int(v))
flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size // 4, dtype=torch.float32, device=dev)
stream = torch.cuda.Stream(dev)
wl.fill()
time_steps(wl, 8, flush, stream)
wl.fill()
ms = np.array(time_steps(wl, K, flush, stream)) * 1e3
by = np.array([wl.shape_at(s).unique_bytes() for s in range(K)], dtype=np.float64)
A = np.stack([np.ones(K), by / 1e6], 1)
(t0, slope), *_ = np.linalg.lstsq(A, ms, rcond=None)
print(f"opts {opts}: mean {ms.mean():.2f} us/step; fit t0 = {t0:.2f} us, rate = {1e6 / slope / 1e3:.0f} GB/s")
for s in [0, 1, 2, 3, 31, 63, 64, 65, 127, 255, 383, 447, 511]:
    if s < K:
        print(f"  step {s:4d}: {ms[s]:6.2f} us  {by[s] / 1e6:7.1f} MB  {by[s] / ms[s] / 1e3:6.0f} GB/s")
