#!/usr/bin/env python
"""Decode-attention benchmark of the B200 ChunkAttention path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--mode chunk|b0|b1] [--workload auto|cfg2|cfg5]

Workload at N = 1 (BASELINE.json configs[1], the metric's configuration):
Llama-2-7B attention shape, 32 heads x 128 dim, fp16, chunk 64, batch 32, a
shared system prompt of 2048 tokens (n_p = n_s = 2048, fully shared,
PAPER.md:348-351), then iterative decoding: a STEP is one decode iteration =
append one token's K/V per sequence (a4, host tree a1-a3) + two-phase
attention (a5 chunk-first, a6 seq-first) for all 32 sequences -- one call of
chunkattn_append_attend, one kernel launch (the K5 cluster decode kernel).
Timed steps are completion tokens 1..K of a fresh cache; token rate = b * K / t
(PAPER.md:348).

Workload at N > 1 (torchrun; BASELINE.json configs[4]): b = 256, shared
prompt 4096, 64-token questions (p = 65 at the first step), the 32 heads split
over the N ranks ("the head dimension is always partitioned"),
every rank replaying the same host op stream; one NCCL all_gather_into_tensor
of the per-rank outputs per step.  Total work is fixed (strong
scaling); value = b * K / max-over-ranks time including the gather.

Timing: CUDA events on the launch stream around each step; the L2 (126 MB on
B200) is flushed between timed steps (outside the events) by writing a 2x-L2
buffer and then reading it back, so L2 holds clean foreign lines.

The JSON line adds: roofline (the K5 kernel's algorithmic bytes / its
per-launch CUDA-event time, against MEASURED_PEAKS.json), seq_first_phase (the
north_star's >= 70 % HBM target: configs[2]'s n_s = 0, b = 32, n_p = 4096
point, K5 and the persistent seq-first kernel), sweep (configs[2] at b = 32:
n_s = 0 / 1024 / 2048 / 4096 with the non-shared paged layout B0 beside it),
p512 (the cfg2 step at 512 private tokens), e2e (wall clock of back-to-back
decode steps through chunkattn_decode_step_host from pinned HOST buffers, one
stream sync per step, plus the host microseconds of the call: tree + context
+ launch), cpu_baseline (the fp64 oracle on the host, all cores and 1 core),
gpu_launches, clocks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "decode attention tokens/s and kernel µs vs shared-prompt len; % HBM roofline"


# ------------------------------------------------------------------ helpers --
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j.get("hbm_gbs", 6650.0), "measured", j
    return 6650.0, "fallback", {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the run."""
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,utilization.gpu")

    def __init__(self, index: int):
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def snapshot(self):
        """Clock statistics of the samples so far (the sampler keeps running)."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.f.flush()
        return self._summary()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        time.sleep(0.05)
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        res = self._summary()
        os.unlink(self.path)
        return res

    def _summary(self):
        sm, mx, reasons = [], None, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    s, m, util = float(parts[1]), float(parts[2]), float(parts[7])
                except ValueError:
                    continue
                mx = m
                if util > 0:
                    sm.append(s)
                for nm, v in zip(names, parts[3:7]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------- workload --
class DecodeWorkload:
    """b sequences sharing a prompt of n_shared tokens (+ optional private
    question), decoded for `steps` iterations; all inputs generated on the device
    before timing (synthetic, seeded; DESIGN.md input recipe)."""

    def __init__(self, dev, seed=0, b=32, h=32, d=128, c=64, n_shared=2048, question=0, steps=512,
                 dtype=torch.float16, mode="chunk"):
        from paper_2402_15220_b200 import ChunkAttention
        self.dev, self.seed, self.b, self.h, self.d, self.c = dev, seed, b, h, d, c
        self.n_shared, self.question, self.steps, self.dtype, self.mode = n_shared, question, steps, dtype, mode
        max_len = n_shared + question + steps + 1
        per_seq = (max_len + c - 1) // c
        max_chunks = per_seq * b + 8 if mode == "b0" else (n_shared // c + 1) + b * ((question + steps) // c + 2)
        thr = (1 << 30) if mode == "b1" else 2
        self.ca = ChunkAttention(h, d, c, max_chunks, b, max_len, dtype=dtype, out_dtype=dtype,
                                 share_threshold=thr, prefix_match=(mode != "b0"), device=dev)
        self.prompt = synth.token_ids(seed, synth.TAG_SYS, 0, n_shared, device=dev)
        self.questions = [synth.token_ids(seed, synth.TAG_PRIV, r, question, device=dev) for r in range(b)]
        pos = torch.arange(n_shared, device=dev)
        self.k_prompt = synth.kv_values(seed, synth.TID_K, self.prompt, pos, 1, h, d, device=dev).to(dtype)
        self.v_prompt = synth.kv_values(seed, synth.TID_V, self.prompt, pos, 1, h, d, device=dev).to(dtype)
        # per-step decode inputs, resident in HBM: tokens, k/v [S][b][1][h][d], q [S][b][h][d]
        S = steps
        rows = torch.arange(b, device=dev, dtype=torch.int64)
        st = torch.arange(S, device=dev, dtype=torch.int64)
        tok = 1 + synth.hash_keys(seed, synth.TAG_DECODE, rows[None, :], st[:, None], device=dev) % 31999
        self.tokens = tok.to(torch.int32).cpu().numpy()                        # [S][b]
        self.kn = torch.empty((S, b, 1, h, d), dtype=dtype, device=dev)
        self.vn = torch.empty_like(self.kn)
        self.q = torch.empty((S, b, h, d), dtype=dtype, device=dev)
        base = n_shared + question
        for s in range(S):
            p = torch.full((b,), base + s, dtype=torch.int64, device=dev)
            t = tok[s]
            self.kn[s] = synth.kv_values(seed, synth.TID_K, t, p, 1, h, d, device=dev).to(dtype)
            self.vn[s] = synth.kv_values(seed, synth.TID_V, t, p, 1, h, d, device=dev).to(dtype)
        for s0 in range(0, S, 64):
            s1 = min(S, s0 + 64)
            for s in range(s0, s1):
                self.q[s] = synth.q_values(seed, rows, s + 1, 1, h, d, alpha=8.0, device=dev)[:, 0].to(dtype)
        self.out = torch.empty((b, h, d), dtype=dtype, device=dev)
        self.ids = None
        self.one_launch = True

    def fill(self):
        """Drain the cache and insert the b sequences (prefill with prefix lookup)."""
        if self.ids is not None:
            for s in self.ids.tolist():
                self.ca.remove_sequence(s)
        ids = []
        for r in range(self.b):
            toks = torch.cat([self.prompt, self.questions[r]]).tolist()
            m = self.ca.match_prefix(toks)
            pos = torch.arange(m, len(toks), device=self.dev)
            if m < self.n_shared:
                k = torch.cat([self.k_prompt[m:], self._qkv(synth.TID_K, r)])
                v = torch.cat([self.v_prompt[m:], self._qkv(synth.TID_V, r)])
            else:
                k = self._qkv(synth.TID_K, r, m - self.n_shared)
                v = self._qkv(synth.TID_V, r, m - self.n_shared)
            assert k.shape[0] == len(pos)
            sid, _ = self.ca.add_sequence(toks, k.contiguous(), v.contiguous(), kv_first_pos=m)
            ids.append(sid)
        self.ids = np.asarray(ids, dtype=np.int64)
        torch.cuda.synchronize(self.dev)

    def _qkv(self, which, r, skip=0):
        t = self.questions[r][skip:]
        pos = torch.arange(self.n_shared + skip, self.n_shared + self.question, device=self.dev)
        return synth.kv_values(self.seed, which, t, pos, 1, self.h, self.d, device=self.dev).to(self.dtype)

    def step(self, s: int, stream: int):
        if self.one_launch:  # append + attend in one call (one kernel launch with the K5 decode kernel)
            self.ca.append_attend_raw(self.ids, self.tokens[s], self.kn[s].data_ptr(), self.vn[s].data_ptr(),
                                      self.q[s].data_ptr(), self.out.data_ptr(), stream)
            return
        self.ca.append_raw(self.ids, self.tokens[s], self.kn[s].data_ptr(), self.vn[s].data_ptr(), stream)
        self.ca.attend_raw(0, self.ids, self.q[s].data_ptr(), self.out.data_ptr(), stream)

    def shape_at(self, s: int):
        """StepShape of decode step s (0-based): private tokens per row = question + s + 1."""
        from paper_2402_15220_b200.roofline import StepShape
        p = self.question + s + 1
        if self.mode == "chunk":
            shared = self.n_shared // self.c
            priv = self.b * (p + self.n_shared % self.c)
            return StepShape(self.b, self.h, self.d, self.c, 2, 2, shared, shared * self.b,
                             self.b if shared else 0, priv)
        # baselines: no chunk-first phase; every row walks its whole context
        return StepShape(self.b, self.h, self.d, self.c, 2, 2, 0, 0, 0, self.b * (self.n_shared + p))


# -------------------------------------------------------------------- arms --
def flush_l2(buf):
    """Evict L2 between timed steps: write a 2x-L2 buffer, then read it back so
    the lines left in L2 are clean (otherwise the timed step would also pay
    the HBM write-back of ~L2-size of the flush buffer's dirty lines).  Our
    inputs are not L2-resident either way."""
    buf.zero_()
    buf.sum()


def time_steps(wl: DecodeWorkload, K: int, flush_buf, stream, s0: int = 0) -> list[float]:
    sp = stream.cuda_stream
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with torch.cuda.stream(stream):
        for s in range(K):
            flush_l2(flush_buf)
            evs[s][0].record(stream)
            wl.step(s0 + s, sp)
            evs[s][1].record(stream)
    stream.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def time_e2e_wall(wl: DecodeWorkload, K: int, stream):
    """Same steps through the C ABI with HOST buffers
    (chunkattn_decode_step_host), back to back as a serving loop runs them:
    every step's q, k_new, v_new come from one packed pinned host buffer (one
    H2D inside the call) and its output goes to pinned host memory (one D2H
    inside the call); wall clock (perf_counter) around call + stream sync, no
    L2 flush.  Also the host time of the call alone (tree a1, context a2, lazy
    upload a3, launches)."""
    sp = stream.cuda_stream
    nq, nk = wl.q[0].numel(), wl.kn[0].numel()
    host = torch.empty((K, nq + 2 * nk), dtype=wl.q.dtype).pin_memory()
    host[:, :nq] = wl.q[:K].reshape(K, -1).cpu()
    host[:, nq:nq + nk] = wl.kn[:K].reshape(K, -1).cpu()
    host[:, nq + nk:] = wl.vn[:K].reshape(K, -1).cpu()
    hout = torch.empty((K,) + tuple(wl.out.shape), dtype=wl.out.dtype).pin_memory()
    es = host.element_size()
    staging = torch.empty(((nq + 2 * nk) * es + 15) // 16 * 16 + wl.out.numel() * wl.out.element_size(),
                          dtype=torch.uint8, device=wl.q.device)
    wall, hostcall = [], []
    stream.synchronize()
    for s in range(K):
        t0 = time.perf_counter()
        wl.ca.decode_step_host(wl.ids, wl.tokens[s], host[s], hout[s], staging, stream_ptr=sp)
        t1 = time.perf_counter()
        stream.synchronize()
        t2 = time.perf_counter()
        wall.append(t2 - t0)
        hostcall.append(t1 - t0)
    return wall, hostcall, (nq + 2 * nk) * es, wl.out.numel() * wl.out.element_size()


def cpu_baseline(seed, n_shared, question, h, d, budget_s, max_steps):
    """fp64 oracle on the host: row 0's decode step at completion tokens 1..n
    until the budget is spent (materialisation untimed), with the BLAS pool at
    all host cores and at one core (threadpoolctl)."""
    from threadpoolctl import threadpool_limits

    from oracle.reference import OracleSequence, timed_attend
    prompt = synth.token_ids(seed, synth.TAG_SYS, 0, n_shared).tolist()
    q0 = synth.token_ids(seed, synth.TAG_PRIV, 0, question).tolist()
    ncores = os.cpu_count() or 1
    res = {}
    for label, cores, budget in (("all", ncores, budget_s / 2), ("one", 1, budget_s / 2)):
        seq = OracleSequence(seed, prompt + q0, h, d, n_shared + question + max_steps + 1)
        wall = cpu = 0.0
        n = 0
        t_start = time.perf_counter()
        with threadpool_limits(limits=cores):
            while n < max_steps and time.perf_counter() - t_start < budget:
                tok = int(synth.hash_py(seed, synth.TAG_DECODE, 0, n) % 31999 + 1)
                seq.extend([tok])
                q = synth.q_values(seed, torch.tensor([0]), n + 1, 1, h, d, alpha=8.0)[0, 0].numpy()
                _, w, c = timed_attend(seq, q)
                wall += w
                cpu += c
                n += 1
        res[label] = (n / wall, max(1, round(cpu / wall)), n, wall)
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        model = "unknown"
    v, used, n, wall = res["all"]
    return {"value": v, "unit": "tokens/s", "cores": used, "kind": "oracle",
            "host_cores": ncores, "cpu_model": model, "blas_limit_all_cores": ncores,
            "value_1core": res["one"][0], "cores_1core": 1,
            "sample": f"fp64 numpy oracle (C1), row 0 of the cfg2 batch at completion tokens 1..{n} "
                      f"(context {n_shared + question + 1}..{n_shared + question + n}); attention math only, "
                      f"KV materialisation untimed; {wall:.1f} s (BLAS pool at all {ncores} cores) + "
                      f"{res['one'][3]:.1f} s (1 core) of CPU work; 'cores' = threads the timed run kept busy"}


def kernel_point(dev, flush_buf, stream, K=5, W=3, **kw):
    """Per-kernel CUDA-event time (us per launch) and event-bracketed step time
    of K decode steps of a DecodeWorkload and the algorithmic bytes of those
    steps: completion tokens W+1..W+K of a fresh cache, after W untimed steps
    (the first decode step of a prompt ending on a chunk boundary grows a chunk
    per row -- a structural step whose context rebuild is host work, not the
    steady-state decode step the sweep compares)."""
    opts = kw.pop("opts", {})
    wl = DecodeWorkload(dev, steps=K + W, **kw)
    for k, v in opts.items():
        wl.ca.set_option(k, v)
    if opts.get("dk") == 0:
        wl.one_launch = False
    wl.fill()
    time_steps(wl, W, flush_buf, stream)
    wl.ca.set_option("kernel_events", 1)
    wl.ca.kernel_times()
    ms = time_steps(wl, K, flush_buf, stream, s0=W)
    kt = wl.ca.kernel_times()
    wl.ca.set_option("kernel_events", 0)
    shapes = [wl.shape_at(s) for s in range(W, W + K)]
    attn_ms = kt["seq_first"][0] + kt["chunk_first"][0]
    n_attn = max(1, kt["seq_first"][1])
    res = {"step_us": 1e3 * sum(ms) / K, "attend_kernel_us": 1e3 * attn_ms / n_attn,
           "alg_bytes_per_step": sum(x.unique_bytes() for x in shapes) / K,
           "seq_first_bytes_per_step": sum(x.seq_first_bytes() for x in shapes) / K,
           "sched": wl.ca.schedule_info()}
    del wl
    torch.cuda.empty_cache()
    return res


def extra_points(dev, flush_buf, stream, hbm_peak):
    """The north_star's own checks on the same box: the seq-first-phase HBM
    fraction (configs[2], n_s = 0, b = 32, n_p = 4096), the configs[2] mini sweep
    with B0, the cfg2 step at 512 private tokens."""
    out = {}
    sf = {}
    for label, opts in (("k5", {}), ("persistent_seq_first", {"dk": 0})):
        r = kernel_point(dev, flush_buf, stream, b=32, n_shared=0, question=4095, opts=opts)
        gbs = r["alg_bytes_per_step"] / (r["attend_kernel_us"] * 1e-6) / 1e9
        sf[label] = {"kernel_us": r["attend_kernel_us"], "alg_bytes": r["alg_bytes_per_step"], "achieved": gbs,
                     "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak, "step_us": r["step_us"]}
    sf["workload"] = ("configs[2] n_s = 0, b = 32, n_p = 4096 (4095-token private question + the decode token): "
                      "every byte private, the attention kernel is the sequence-first phase; per-launch CUDA events, "
                      "completion tokens 4..8 (after 3 untimed steps), L2 flushed")
    out["seq_first_phase"] = sf
    sweep = []
    for n_s in (0, 1024, 2048, 4096):
        row = {"n_s": n_s, "n_p": 4096, "b": 32}
        for mode in ("chunk", "b0"):
            r = kernel_point(dev, flush_buf, stream, b=32, n_shared=n_s, question=4096 - n_s, mode=mode)
            row[mode] = {"step_us": r["step_us"], "kernel_us": r["attend_kernel_us"],
                         "alg_bytes": r["alg_bytes_per_step"]}
        row["speedup_vs_b0"] = row["b0"]["kernel_us"] / row["chunk"]["kernel_us"]  # attention kernel per step
        row["step_speedup_vs_b0"] = row["b0"]["step_us"] / row["chunk"]["step_us"]
        row["ideal_bytes_ratio"] = row["b0"]["alg_bytes"] / row["chunk"]["alg_bytes"]
        row["chunk_frac_hbm"] = row["chunk"]["alg_bytes"] / (row["chunk"]["kernel_us"] * 1e-6) / 1e9 / hbm_peak
        sweep.append(row)
    out["sweep"] = sweep
    r = kernel_point(dev, flush_buf, stream, b=32, n_shared=2048, question=511)
    out["p512"] = {"workload": "cfg2 with a 511-token question: p = 512..516 private tokens", "step_us": r["step_us"],
                   "kernel_us": r["attend_kernel_us"], "tokens_per_s": 32 / (r["step_us"] * 1e-6),
                   "frac_hbm": r["alg_bytes_per_step"] / (r["attend_kernel_us"] * 1e-6) / 1e9 / hbm_peak}
    return out


def run_reference(args):
    """`--impl reference`: the oracle as it stands, timed on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.reference import OracleSequence, timed_attend
    h, d, n_shared, seed = 32, 128, 2048, 0
    K, W = args.steps, args.warmup
    prompt = synth.token_ids(seed, synth.TAG_SYS, 0, n_shared).tolist()
    seq = OracleSequence(seed, prompt, h, d, n_shared + W + K + 1)
    times = []
    cpu = 0.0
    for s in range(W + K):
        tok = int(synth.hash_py(seed, synth.TAG_DECODE, 0, s) % 31999 + 1)
        seq.extend([tok])
        q = synth.q_values(seed, torch.tensor([0]), s + 1, 1, h, d, alpha=8.0)[0, 0].numpy()
        _, w, c = timed_attend(seq, q)
        if s >= W:
            times.append(w)
            cpu += c
    tot = sum(times)
    value = K / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": K, "warmup": W, "ms_per_step": 1e3 * tot / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2_llama2_7b_b32_s2048 (oracle: 1 sequence per step)", "b": 32, "h": h,
                       "d": d, "c": 64, "n_shared": n_shared, "l2": "n/a (CPU)"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": max(1, round(cpu / tot)), "kind": "oracle",
                             "sample": f"each step = one sequence's decode attention (fp64 numpy, C1) at context "
                                       f"{n_shared + W + 1}..{n_shared + W + K}; KV materialisation untimed"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_cfg2(args):
    """N = 1: the metric's configuration (BASELINE.json configs[1])."""
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    K, W = args.steps, args.warmup
    hbm_peak, peak_src, _ = load_peaks()
    sampler = ClockSampler(0)
    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 * 2 ** 20) or 126 * 2 ** 20
    flush_buf = torch.empty(2 * l2 // 4 + 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)
    wl = DecodeWorkload(dev, seed=0, steps=max(K, W), mode=args.mode, question=args.question,
                        n_shared=args.n_shared, b=args.batch)
    for o in args.opt:
        key, val = o.split("=")
        wl.ca.set_option(key, int(val))
        if key == "dk" and int(val) == 0:
            wl.one_launch = False
    # warm-up on the same cache, then drain and refill: timed steps are tokens 1..K
    wl.fill()
    time_steps(wl, W, flush_buf, stream)
    t0 = time.time()  # spin the clocks up (~0.3 s of memsets) so the timed region runs at boost
    while time.time() - t0 < 0.3:
        flush_l2(flush_buf)
    torch.cuda.synchronize(dev)
    # ---- pass A: the headline number
    wl.fill()
    c0 = wl.ca.counters()
    torch.cuda.synchronize(dev)
    ms = time_steps(wl, K, flush_buf, stream)
    torch.cuda.synchronize(dev)
    c1 = wl.ca.counters()
    total_ms = sum(ms)
    launches = c1["launches"] - c0["launches"]
    uploads = c1["uploads"] - c0["uploads"]
    sched = wl.ca.schedule_info()
    # ---- pass B: per-kernel CUDA events (roofline of the dominant kernel)
    wl.fill()
    wl.ca.set_option("kernel_events", 1)
    wl.ca.kernel_times()
    ms_b = time_steps(wl, K, flush_buf, stream)
    kt = wl.ca.kernel_times()
    wl.ca.set_option("kernel_events", 0)
    shapes = [wl.shape_at(s) for s in range(K)]
    fused = wl.one_launch and sched["dk"] == 1
    if fused:  # K5: append + both phases + merge in the one kernel
        kbytes = {"append": 0, "chunk_first": 0, "seq_first": sum(x.fused_step_bytes() for x in shapes)}
        kname = "dk_kernel (K5 cluster decode: append + chunk-first + seq-first + cluster merge)"
    else:
        kbytes = {"append": sum(x.append_bytes() for x in shapes),
                  "chunk_first": sum(x.chunk_first_bytes() for x in shapes),
                  "seq_first": sum(x.seq_first_bytes() for x in shapes)}
        if kt["chunk_first"][1] == 0:  # fused persistent kernel runs the chunk-first units too
            kbytes["seq_first"] = sum(x.unique_bytes() for x in shapes)
            kbytes["chunk_first"] = 0
        kname = "sf_persistent_kernel"
    dom = max(("append", "chunk_first", "seq_first"), key=lambda k: kt[k][0])
    dom_ms, dom_n = kt[dom]
    achieved = kbytes[dom] / (dom_ms * 1e-3) / 1e9 if dom_ms > 0 else None
    traffic, traffic_note = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f).get(f"{args.mode}:{'k5' if fused else dom}")
        if isinstance(tr, dict):  # one ncu --set full launch of a timed step: its DRAM bytes vs algorithmic
            traffic = tr.get("bytes")
            traffic_note = {"alg_bytes_same_launch": tr.get("alg_bytes"), "decode_step": tr.get("step"),
                            "capture": tr.get("capture")}
    kernels = {k: {"ms_total": kt[k][0], "launches": kt[k][1],
                   "us_avg": 1e3 * kt[k][0] / kt[k][1] if kt[k][1] else None,
                   "alg_bytes_per_launch": kbytes[k] / kt[k][1] if kt[k][1] else None,
                   "gbs": kbytes[k] / (kt[k][0] * 1e-3) / 1e9 if kt[k][0] else None}
               for k in ("append", "chunk_first", "seq_first")}
    step_bytes = sum(x.unique_bytes() for x in shapes)
    # ---- pass C: end to end through the C ABI with host buffers (wall clock)
    wl.fill()
    time_e2e_wall(wl, min(W, K), stream)  # warm the host path
    wl.fill()
    wall, hostcall, h2d, d2h = time_e2e_wall(wl, K, stream)
    del wl
    torch.cuda.empty_cache()
    # ---- the north_star's own checks (seq-first HBM fraction, sweep vs B0, p = 512)
    extras = {} if args.no_extras else extra_points(dev, flush_buf, stream, hbm_peak)
    clocks = sampler.stop()
    value = args.batch * K / (total_ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": 1, "steps": K, "warmup": W,
        "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f16", "data": "synthetic",
        "config": {"workload": f"cfg2_llama2_7b_b{args.batch}_s{args.n_shared}" + ("" if args.mode == "chunk" else f"_{args.mode}"),
                   "b": args.batch, "h": 32, "d": 128, "c": 64, "n_shared": args.n_shared,
                   "question": args.question, "completion_tokens_timed": f"1..{K}", "mode": args.mode,
                   "step": "chunkattn_append_attend (one K5 launch)" if fused else "append_kv + attend",
                   "schedule": sched,
                   "l2": "flushed between timed steps (write a 2x-L2 buffer, then read it back so L2 holds clean "
                         "foreign lines; outside the events)",
                   "parallelism": "1 GPU"},
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak if achieved else None, "traffic": traffic,
                     "traffic_note": traffic_note, "peak_source": peak_src,
                     "avg_launch_us": 1e3 * dom_ms / dom_n if dom_n else None,
                     "alg_bytes_per_launch": kbytes[dom] / dom_n if dom_n else None,
                     "bytes_model": "every distinct K/V element once (the new row from the caller's k/v) + q + o "
                                    "+ the new rows' pool writes (roofline.StepShape.fused_step_bytes)"},
        "kernels": kernels,
        "step_unique_bytes_avg": step_bytes / K,
        "step_gbs_vs_unique_bytes": step_bytes / (total_ms * 1e-3) / 1e9,
        "passB_ms_per_step": sum(ms_b) / K,
        "uploads_in_timed_region": uploads,
        "e2e": {"value": args.batch * K / sum(wall), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * sum(wall) / K,
                "host_us_per_step": 1e6 * statistics.median(hostcall),
                "host_us_per_step_mean": 1e6 * sum(hostcall) / K,
                "method": "wall clock (perf_counter) of back-to-back chunkattn_decode_step_host calls, each followed "
                          "by a stream sync: packed pinned host [q|k_new|v_new] -> one H2D, the K5 step, one D2H "
                          "to pinned host; no L2 flush. host_us = the call alone (tree a1 + context a2 + lazy "
                          "upload a3 + launches, Python/ctypes included)"},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    line.update(extras)
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(0, args.n_shared, args.question, 32, 128, args.cpu_budget, 4096)
    print(json.dumps(line), flush=True)


def run_sharded(args):
    """BASELINE.json configs[4] over the N ranks of one node: b = 256, shared
    prompt 4096, 64-token questions; rank r holds heads [r h/N, (r+1) h/N) and
    replays the full host op stream; each step = append_attend on the local
    heads + one all_gather_into_tensor of the outputs (+ the head permutation)."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = args.dist_backend
    if world > 1:
        dist.init_process_group(backend)
    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local % ndev)
    torch.cuda.set_device(dev)
    K, W = args.steps, args.warmup
    H, b = 32, args.batch_cfg5
    if H % world:
        raise SystemExit(f"{H} heads do not split over {world} ranks")
    hl = H // world
    hbm_peak, peak_src, _ = load_peaks()
    sampler = ClockSampler(local % ndev) if rank == 0 else None
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.empty(2 * l2 // 4 + 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)
    # every rank: the same host op stream (same seed), its heads' K/V only
    wl = DecodeWorkload(dev, seed=0, steps=max(K, W), b=b, h=hl, n_shared=4096, question=64)
    gbuf = torch.empty((world, b, hl, 128), dtype=torch.float16, device=dev)

    def gather():
        if world == 1:
            return wl.out
        if backend == "nccl":
            dist.all_gather_into_tensor(gbuf, wl.out)
        else:  # gloo (CPU-side test of the path): staged through the host
            parts = [torch.empty((b, hl, 128), dtype=torch.float16) for _ in range(world)]
            dist.all_gather(parts, wl.out.cpu())
            gbuf.copy_(torch.stack(parts))
        return gbuf.permute(1, 0, 2, 3).reshape(b, H, 128)

    def steps_timed(n, with_gather):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        with torch.cuda.stream(stream):
            for s in range(n):
                flush_l2(flush_buf)
                evs[s][0].record(stream)
                wl.step(s, stream.cuda_stream)
                if with_gather:
                    gather()
                evs[s][1].record(stream)
        stream.synchronize()
        return [a.elapsed_time(z) for a, z in evs]

    wl.fill()
    steps_timed(W, True)
    wl.fill()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ms_g = steps_timed(K, True)
    wl.fill()
    ms_k = steps_timed(K, False)
    tot = torch.tensor([sum(ms_g), sum(ms_k)], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        dist.barrier()
    total_g, total_k = float(tot[0]), float(tot[1])
    shapes = [wl.shape_at(s) for s in range(K)]
    bytes_rank = sum(x.fused_step_bytes() for x in shapes) / K
    sched = wl.ca.schedule_info()
    clocks = sampler.stop() if sampler else None
    if rank == 0:
        line = {
            "metric": METRIC, "value": b * K / (total_g * 1e-3), "unit": "tokens/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": total_g / K, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f16", "data": "synthetic",
            "config": {"workload": "cfg5_b256_s4096_q64_head_sharded", "b": b, "h": H, "heads_per_rank": hl,
                       "d": 128, "c": 64, "n_shared": 4096, "question": 64, "completion_tokens_timed": f"1..{K}",
                       "parallelism": f"heads split over {world} ranks (tp{world}); one {backend} "
                                      f"all_gather_into_tensor of the outputs per step",
                       "schedule_rank0": sched,
                       "l2": "flushed between timed steps (outside the events)"},
            "kernel_only_ms_per_step": total_k / K,
            "gather_ms_per_step": (total_g - total_k) / K,
            "roofline": {"bound": "hbm", "kernel": "dk_kernel (K5), per rank", "achieved":
                         bytes_rank / (total_k / K * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                         "frac": bytes_rank / (total_k / K * 1e-3) / 1e9 / hbm_peak, "traffic": None,
                         "peak_source": peak_src, "alg_bytes_per_launch_per_rank": bytes_rank,
                         "note": "event time of the whole step (launch included) per rank, max over ranks"},
            "e2e": {"value": b * K / (total_g * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0, "note": "device-resident inputs on the sharded path"},
            "gpu_launches": K,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_ours(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    workload = args.workload
    if workload == "auto":
        workload = "cfg5" if world > 1 else "cfg2"
    if workload == "cfg5":
        run_sharded(args)
    else:
        if world > 1:
            raise SystemExit("cfg2 is a one-GPU workload; use --workload cfg5 (the sharded configs[4])")
        run_cfg2(args)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=512)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="chunk", choices=["chunk", "b0", "b1"])
    ap.add_argument("--n-shared", dest="n_shared", type=int, default=2048)
    ap.add_argument("--question", type=int, default=0)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--cpu-budget", dest="cpu_budget", type=float, default=16.0)
    ap.add_argument("--no-cpu", dest="no_cpu", action="store_true")
    ap.add_argument("--opt", action="append", default=[], help="library option key=value (A/B experiments)")
    ap.add_argument("--workload", default="auto", choices=["auto", "cfg2", "cfg5"],
                    help="auto: cfg2 on one GPU (the metric's config), the head-sharded cfg5 under torchrun")
    ap.add_argument("--batch-cfg5", dest="batch_cfg5", type=int, default=256)
    ap.add_argument("--dist-backend", dest="dist_backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--no-extras", dest="no_extras", action="store_true",
                    help="skip the seq-first / sweep / p512 points")
    args = ap.parse_args()
    if os.environ.get("CA_BENCH_WATCHDOG"):  # debugging: dump the Python stacks if a pass stalls
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["CA_BENCH_WATCHDOG"]), exit=True)
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
