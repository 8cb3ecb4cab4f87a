"""Debug helper: two-level tree at step 1, fused vs non-fused outputs."""
import random, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from tests.gpu_workload import Harness, decode_tokens

def build(opts):
    rng = random.Random(21)
    c = 16
    hs = Harness(4, 64, c, "f16", "f16", seed=21, alpha=8.0, max_chunks=600)
    for k, v in opts.items():
        hs.ca.set_option(k, v)
    sys_p = synth.token_ids(21, synth.TAG_SYS, 0, 64).tolist()
    groups = [synth.token_ids(21, synth.TAG_GROUP, g, 64).tolist() for g in range(4)]
    live = []
    for k in range(16):
        g = rng.randrange(4)
        q = synth.token_ids(21, synth.TAG_PRIV, k, rng.randint(1, c - 1)).tolist()
        live.append(hs.add(sys_p + groups[g] + q)[0])
        rng.randint(8, 60)
    hs.step = 1
    hs.append(live, decode_tokens(hs, live))
    return hs, live

a, live = build({"fused": 1})
b, _ = build({"fused": 0})
q64 = a.queries(live)
oa = a.ca.attend(live, q64.to(a.dev, a.dt).contiguous()).double().cpu()
ob = b.ca.attend(live, q64.to(b.dev, b.dt).contiguous()).double().cpu()
ref = a.oracle(live, q64)
err_a = (oa.numpy() - ref).__abs__().max(-1)
err_b = (ob.numpy() - ref).__abs__().max(-1)
print("fused bad:", np.argwhere(err_a > 2e-3).tolist())
print("nonfused bad:", np.argwhere(err_b > 2e-3).tolist())
print("order:", a.ca.batch_order())
print("live (caller order):", live)
print(a.ca.export_context())
