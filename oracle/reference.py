"""Oracle decode step for bench.py's CPU legs — TEST INFRASTRUCTURE ONLY.

bench.py's `cpu_baseline` (rank 0, N = 1) and its `--impl reference` arm time
exactly this: the C1 oracle (attention.attend_heads_fp64, the plain
softmax(s q K^T) V of PAPER.md:344 over one sequence's materialised, unshared
KV) for one decode step of one sequence.  The KV
materialisation from the seeded generator is NOT timed; only the attention
arithmetic is.  Nothing here is tuned.
"""
from __future__ import annotations

import time

import numpy as np
import torch

import synth
from .attention import attend_heads_fp64, default_scale


class OracleSequence:
    """One sequence's fully materialised fp64 K/V (layer 0), grown per decode step."""

    def __init__(self, seed: int, tokens, h: int, d: int, max_len: int):
        self.seed, self.h, self.d = seed, h, d
        self.K = np.zeros((max_len, h, d))
        self.V = np.zeros((max_len, h, d))
        self.n = 0
        self.extend(tokens)

    def extend(self, tokens):
        t = torch.as_tensor(list(tokens), dtype=torch.int64)
        pos = torch.arange(self.n, self.n + len(t), dtype=torch.int64)
        self.K[self.n:self.n + len(t)] = synth.kv_values(self.seed, synth.TID_K, t, pos, 1, self.h, self.d)[:, 0].numpy()
        self.V[self.n:self.n + len(t)] = synth.kv_values(self.seed, synth.TID_V, t, pos, 1, self.h, self.d)[:, 0].numpy()
        self.n += len(t)

    def attend(self, q):
        return attend_heads_fp64(q, self.K[:self.n], self.V[:self.n], default_scale(self.d))


def timed_attend(seq: OracleSequence, q) -> tuple[np.ndarray, float, float]:
    """(output, wall seconds, process CPU seconds) of one oracle decode step."""
    w0, c0 = time.perf_counter(), time.process_time()
    o = seq.attend(q)
    return o, time.perf_counter() - w0, time.process_time() - c0
