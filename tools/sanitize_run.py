"""Small decode workloads for compute-sanitizer (memcheck / racecheck /
synccheck): the tiny config (configs[0], fp16), a small c = 64 tree on both K5
variants (chunk-first units on tcgen05 and on mma.sync) and one cfg2 step, on
the K5 one-launch path and on the persistent kernels (dk=0: fused and
two-kernel), each checked against the fp64 oracle so a silent corruption also
fails.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [--cfg2]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.gpu_workload import Harness, build_shared, decode_tokens  # noqa: E402

variants = ["", "dk=0", "dk=0,fused=0"]
for opts in variants:
    hs = Harness(8, 64, 16, "f16", "f16", seed=1, alpha=8.0, opts=opts)
    ids = build_shared(hs, 64, [0, 1, 16, 32])
    hs.check(ids, 2e-3)
    for st in range(1, 3):
        hs.step = st
        hs.append_attend(ids, decode_tokens(hs, ids), 2e-3)
    print("tiny ok", opts or "K5", flush=True)
for opts in ["dk_umma=2", "dk_umma=0", "dk_umma=2,dk_cs=2"]:  # c = 64: the tcgen05 chunk-first variant
    hs = Harness(4, 128, 64, "f16", "f16", seed=2, alpha=8.0, opts=opts)
    ids = build_shared(hs, 256, [0, 5, 64, 70, 1, 130])
    hs.check(ids, 2e-3)
    for st in range(1, 3):
        hs.step = st
        hs.append_attend(ids, decode_tokens(hs, ids), 2e-3)
    print("c64 ok", opts, flush=True)
if "--cfg2" in sys.argv:
    for opts in variants + ["dk_umma=0"]:
        hs = Harness(32, 128, 64, "f16", "f16", seed=3, alpha=8.0, max_chunks=512, opts=opts)
        ids = build_shared(hs, 2048, [0] * 32)
        hs.step = 1
        hs.append_attend(ids, decode_tokens(hs, ids), 2e-3, rows=[0, 31])
        print("cfg2 ok", opts or "K5", flush=True)
