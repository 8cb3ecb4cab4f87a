"""Serving-loop workload over the library (PAPER.md:49
iteration-based batching, "new sequences can join, and completed sequences
can leave"; PAPER.md:447-449 Poisson arrivals, normalised latency and peak
KV-cache bytes; PAPER.md:511 the 1/(1 - r) capacity argument).

There are no model weights here: an iteration runs exactly the attention work
of the method -- prefill attention with prefix lookup for the requests that
join (chunkattn_add_sequence + chunkattn_prefill_attend) and one decode step
for the running batch (chunkattn_append_attend: one launch) -- on seeded
synthetic K/V/Q (synth/).  The clock advances by each iteration's device time
(CUDA events around the iteration's launches), so latencies are attention-only;
on a host-only handle (no GPU) it advances by a fixed cost per iteration.  The
KV-memory metrics come from chunkattn_memory_stats and are exact.

Everything that moves data runs in the CUDA library; this module only decides
who joins, who leaves, and which tokens / rows are passed (argument
marshalling around the C ABI calls).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

import synth

from .attention import ChunkAttention


@dataclass
class Request:
    rid: int
    arrival_s: float
    prompt: list[int]
    n_c: int


@dataclass
class RunMetrics:
    mode: str
    requests: int
    completion_tokens: int
    normalized_latency_ms_per_tok: float   # mean over requests of (finish - arrival) / n_c
    mean_latency_ms: float
    makespan_ms: float
    peak_batch: int
    peak_kv_chunks: int
    peak_kv_bytes: int
    prefill_tokens_computed: int           # queries (and K/V rows) actually computed in prefill
    prefill_tokens_matched: int            # prompt tokens served by prefix lookup
    iterations: int
    latencies_ms: list[float] = field(default_factory=list, repr=False)


def poisson_trace(seed: int, n_requests: int, rps: float, n_p: int, n_s: int, n_c: int) -> list[Request]:
    """n_requests arrivals with exponential inter-arrival times (rate rps); every
    prompt = the same n_s-token system prompt + (n_p - n_s) private tokens."""
    rng = np.random.default_rng(seed)
    t = np.cumsum(rng.exponential(1.0 / rps, n_requests)) if rps > 0 else np.zeros(n_requests)
    sys_prompt = synth.token_ids(seed, synth.TAG_SYS, 0, n_s).tolist()
    return [Request(i, float(t[i]), sys_prompt + synth.token_ids(seed, synth.TAG_PRIV, i, n_p - n_s).tolist(), n_c)
            for i in range(n_requests)]


class ServingLoop:
    """Iteration-based batching (admit up to b_max, prefill the joiners, one
    decode step for everyone, retire finished requests) on one FRESH handle."""

    def __init__(self, ca: ChunkAttention, b_max: int, seed: int = 0, host_iter_ms: float = 1.0):
        self.ca, self.b_max, self.seed = ca, b_max, seed
        self.gpu = ca.device is not None and ca.device.type == "cuda"
        self.host_iter_ms = host_iter_ms

    def _kv(self, which, toks, pos):
        dev = self.ca.device if self.gpu else "cpu"
        t = torch.as_tensor(toks, dtype=torch.int64, device=dev)
        p = torch.as_tensor(pos, dtype=torch.int64, device=dev)
        return synth.kv_values(self.seed, which, t, p, self.ca.L, self.ca.h, self.ca.d, device=dev).to(self.ca.dtype)

    def run(self, trace: list[Request], mode: str, observer=None) -> RunMetrics:
        """observer (tests): called after every iteration with a dict of that
        iteration's prefill (ids, first positions, q, out) and decode (ids,
        tokens appended, q, out) and the token lists of the running sequences."""
        ca, gpu = self.ca, self.gpu
        pending = sorted(trace, key=lambda r: r.arrival_s)
        running: dict[int, dict] = {}   # seq id -> {req, tokens, generated}
        clock_ms = 0.0
        lat, peak_b, peak_chunks, peak_bytes = [], 0, 0, 0
        computed = matched_total = iters = 0
        stream = torch.cuda.current_stream(ca.device) if gpu else None
        sid_counter = 0  # a fresh handle: chunkattn_add_sequence ids are 0, 1, 2, ...
        while pending or running:
            if not running and pending and pending[0].arrival_s * 1e3 > clock_ms:
                clock_ms = pending[0].arrival_s * 1e3          # idle until the next arrival
            joiners = []
            while pending and pending[0].arrival_s * 1e3 <= clock_ms and len(running) + len(joiners) < self.b_max:
                joiners.append(pending.pop(0))
            # ---- inputs of this iteration (synthetic, outside the timed region).
            # Sequence ids are monotone (chunkattn_add_sequence), so joiners' ids
            # are known before the calls.
            plan = []
            for j, r in enumerate(joiners):
                plan.append([r, sid_counter + j, None])
            dec_sids = list(running) + [sid_counter + j for j in range(len(joiners))]
            dec_len = [len(running[s]["tokens"]) for s in running] + [len(r.prompt) for r in joiners]
            dec_gen = [running[s]["generated"] for s in running] + [0] * len(joiners)
            toks = [int(synth.hash_py(self.seed, synth.TAG_DECODE, s, g) % 31999 + 1) for s, g in zip(dec_sids, dec_gen)]
            kd = vd = qd = None
            if gpu:
                kd = self._kv(synth.TID_K, toks, dec_len).contiguous()
                vd = self._kv(synth.TID_V, toks, dec_len).contiguous()
                qd = synth.q_values(self.seed, torch.tensor(dec_sids, device=ca.device), iters + 1, 1, ca.h, ca.d,
                                    device=ca.device)[:, 0].to(ca.dtype).contiguous()
                # prompt K/V of every joiner (full prompt: the matched rows are skipped by offset)
                for p_ in plan:
                    r = p_[0]
                    p_.append(self._kv(synth.TID_K, r.prompt, list(range(len(r.prompt)))))
                    p_.append(self._kv(synth.TID_V, r.prompt, list(range(len(r.prompt)))))
                    p_.append(synth.q_values(self.seed, torch.arange(len(r.prompt), device=ca.device) + 7919 * p_[1],
                                             0, 1, ca.h, ca.d, device=ca.device)[:, 0].to(ca.dtype))
                torch.cuda.synchronize(ca.device)
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record(stream)
            # ---- timed: prefill with prefix lookup, then one decode step
            ids, firsts, qs = [], [], []
            for p_ in plan:
                r, want = p_[0], p_[1]
                m = ca.match_prefix(r.prompt)
                k = v = None
                if gpu:
                    k, v = p_[3][m:].contiguous(), p_[4][m:].contiguous()
                sid, got = ca.add_sequence(r.prompt, k, v, kv_first_pos=m)
                if sid != want:
                    raise RuntimeError(f"sequence id {sid} != expected {want}")
                running[sid] = {"req": r, "tokens": list(r.prompt), "generated": 0}
                computed += len(r.prompt) - got
                matched_total += got
                ids.append(sid)
                firsts.append(got)
                if gpu:
                    qs.append(p_[5][got:])
            sid_counter += len(plan)
            pf_out = pf_q = None
            if gpu and ids and sum(q.shape[0] for q in qs) > 0:
                pf_q = torch.cat(qs).contiguous()
                pf_out = ca.prefill_attend(ids, firsts, pf_q)
            if gpu:  # one decode step: append + attend in one call (one K5 launch)
                dec_out = ca.append_attend(dec_sids, toks, kd[:, 0].contiguous(), vd[:, 0].contiguous(), qd)
            else:
                ca.append_kv(dec_sids, toks, kd, vd)
                ca.attend(dec_sids, qd)
                dec_out = None
            if gpu:
                ev1.record(stream)
                ev1.synchronize()
                clock_ms += ev0.elapsed_time(ev1)
            else:
                clock_ms += self.host_iter_ms
            st = ca.memory_stats()
            peak_chunks = max(peak_chunks, st["used"])
            peak_bytes = max(peak_bytes, st["kv_bytes"])
            peak_b = max(peak_b, len(dec_sids))
            iters += 1
            for s, t in zip(dec_sids, toks):
                running[s]["tokens"].append(t)
                running[s]["generated"] += 1
            if observer is not None:
                observer({"iteration": iters, "prefill_ids": ids, "prefill_first": firsts, "prefill_q": pf_q,
                          "prefill_out": pf_out, "decode_ids": list(dec_sids), "decode_q": qd, "decode_out": dec_out,
                          "tokens": {s: list(running[s]["tokens"]) for s in dec_sids}})
            for s in dec_sids:
                if running[s]["generated"] >= running[s]["req"].n_c:
                    r = running.pop(s)["req"]
                    lat.append((clock_ms - r.arrival_s * 1e3, r.n_c))
                    ca.remove_sequence(s)
        n_c_total = sum(r.n_c for r in trace)
        norm = float(np.mean([l / nc for l, nc in lat])) if lat else 0.0
        mean = float(np.mean([l for l, _ in lat])) if lat else 0.0
        return RunMetrics(mode, len(trace), n_c_total, norm, mean, clock_ms, peak_b, peak_chunks, peak_bytes, computed,
                          matched_total, iters, [l for l, _ in lat])
