"""Drive the bench workload to decode step N (for an ncu capture of that step's
kernels):  ncu --set full -k regex:sf_persistent -s N -c 1 python tools/profile_step.py --step N"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import DecodeWorkload, flush_l2, time_steps  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--step", type=int, default=300)
ap.add_argument("--opt", action="append", default=[])
args = ap.parse_args()
dev = torch.device("cuda", 0)
wl = DecodeWorkload(dev, steps=args.step + 2)
for o in args.opt:
    k, v = o.split("=")
    wl.ca.set_option(k, int(v))
flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size // 4, dtype=torch.float32, device=dev)
stream = torch.cuda.Stream(dev)
wl.fill()
time_steps(wl, args.step + 1, flush, stream)
torch.cuda.synchronize()
