"""Host enqueue cost per decode step vs GPU time (is the bench host-bound?)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import DecodeWorkload, flush_l2, time_steps

dev = torch.device("cuda", 0)
K = 256
wl = DecodeWorkload(dev, steps=K)
flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size // 4, dtype=torch.float32, device=dev)
stream = torch.cuda.Stream(dev)
for ev in (0, 1):
    wl.ca.set_option("kernel_events", ev)
    for fl in (1, 0):
        wl.fill()
        sp = stream.cuda_stream
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            for s in range(K):
                if fl:
                    flush_l2(flush)
                evs[s][0].record(stream)
                wl.step(s, sp)
                evs[s][1].record(stream)
        t1 = time.perf_counter()
        stream.synchronize()
        t2 = time.perf_counter()
        gpu = sum(a.elapsed_time(b) for a, b in evs) / K * 1e3
        kt = wl.ca.kernel_times()
        print(f"kernel_events={ev} flush={fl}: host enqueue {1e6 * (t1 - t0) / K:.1f} us/step, wall {1e6 * (t2 - t0) / K:.1f} "
              f"us/step, GPU step events {gpu:.1f} us" + (f", kernels {{{', '.join(f'{k}: {1e3 * v[0] / max(1, v[1]):.1f}' for k, v in kt.items())}}}" if ev else ""))
