"""Repeat the bench's pass A (512 PDL-chained decode steps, L2 flush between)
R times under a given option set; print how many repetitions completed.
    python tools/pdl_stress.py R key=value ...   (one process per option set)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import DecodeWorkload, time_steps

R = int(sys.argv[1])
opts = [o.split("=") for o in sys.argv[2:]]
dev = torch.device("cuda", 0)
wl = DecodeWorkload(dev, steps=512)
for k, v in opts:
    wl.ca.set_option(k, int(v))
flush = torch.empty(64 * 2 ** 20, dtype=torch.float32, device=dev)
stream = torch.cuda.Stream(dev)
ok = 0
try:
    for r in range(R):
        wl.fill()
        ms = time_steps(wl, 512, flush, stream)
        ok += 1
    print("OPTS", sys.argv[2:], "ok", ok, "of", R, "us/step %.1f" % (1e3 * sum(ms) / len(ms)), flush=True)
except Exception as e:
    print("OPTS", sys.argv[2:], "FAILED after", ok, "of", R, str(e).splitlines()[0], flush=True)
