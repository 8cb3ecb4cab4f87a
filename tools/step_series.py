"""Per-step GPU times of the bench's pass A (to find slow structural steps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from bench import DecodeWorkload, time_steps

K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
dev = torch.device("cuda", 0)
wl = DecodeWorkload(dev, steps=K)
flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size // 4, dtype=torch.float32, device=dev)
stream = torch.cuda.Stream(dev)
wl.fill()
time_steps(wl, 8, flush, stream)
wl.fill()
c0 = wl.ca.counters()
ms = np.array(time_steps(wl, K, flush, stream)) * 1e3
c1 = wl.ca.counters()
print("counters delta:", {k: c1[k] - c0[k] for k in c1})
print("mean %.1f us; slowest steps:" % ms.mean(), [(int(i), round(float(ms[i]), 1)) for i in np.argsort(-ms)[:12]])
print("steps 58..70:", [round(float(x), 1) for x in ms[58:71]])
print("steps 0..8:", [round(float(x), 1) for x in ms[0:9]])
