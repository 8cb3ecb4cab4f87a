"""Test helper: drive ChunkAttention with seeded synthetic sequences and
compute the fp64 oracle on the same inputs.  (Test infrastructure: may import
oracle/; the product package never does.)"""
from __future__ import annotations

import os

import numpy as np
import torch

import synth
from oracle.attention import attend_heads_fp64, default_scale
from paper_2402_15220_b200 import ChunkAttention

TORCH_DT = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}


class Harness:
    """Keeps the token lists of live sequences so the oracle can regenerate
    every sequence's KV (KV depends only on (token, position))."""

    def __init__(self, h, d, c, dtype="f16", out_dtype=None, num_layers=1, seed=0, alpha=1.0, mode="chunk",
                 max_chunks=4096, max_batch=256, max_seq_len=8192, kv_fn=None, device="cuda", opts=""):
        self.h, self.d, self.c, self.L = h, d, c, num_layers
        self.dt = TORCH_DT[dtype]
        self.odt = TORCH_DT[out_dtype or dtype]
        self.seed, self.alpha = seed, alpha
        self.kv_fn = kv_fn or self._kv_synth
        self.custom_kv = kv_fn is not None
        thr = (1 << 30) if mode == "b1" else 2
        self.ca = ChunkAttention(h, d, c, max_chunks, max_batch, max_seq_len, dtype=self.dt, out_dtype=self.odt,
                                 num_layers=num_layers, share_threshold=thr, prefix_match=(mode != "b0"),
                                 device=device)
        self.dev = self.ca.device
        # library options ("key=value,..."): the test's own, then CA_TEST_OPTS
        for kv in filter(None, (opts + "," + os.environ.get("CA_TEST_OPTS", "")).split(",")):
            key, val = kv.split("=")
            self.ca.set_option(key, int(val))
        self.seqs: dict[int, list[int]] = {}
        self.step = 0

    def _kv_synth(self, which, toks, pos):
        return synth.kv_values(self.seed, which, toks, pos, self.L, self.h, self.d, device=self.dev)

    def kv(self, toks, pos):
        """float64 K, V [n][L][h][d] (on the GPU for the default generator)."""
        dev = "cpu" if self.custom_kv else self.dev
        t = torch.as_tensor(toks, dtype=torch.int64, device=dev)
        p = torch.as_tensor(pos, dtype=torch.int64, device=dev)
        return self.kv_fn(synth.TID_K, t, p), self.kv_fn(synth.TID_V, t, p)

    def add(self, toks, kv_first_pos=0):
        k, v = self.kv(toks[kv_first_pos:], list(range(kv_first_pos, len(toks))))
        sid, m = self.ca.add_sequence(toks, k.to(self.dev, self.dt).contiguous(), v.to(self.dev, self.dt).contiguous(),
                                      kv_first_pos=kv_first_pos)
        self.seqs[sid] = list(toks)
        return sid, m

    def remove(self, sid):
        del self.seqs[sid]
        return self.ca.remove_sequence(sid)

    def append(self, ids, toks):
        pos = [len(self.seqs[s]) for s in ids]
        k, v = self.kv(toks, pos)
        self.ca.append_kv(ids, toks, k.to(self.dev, self.dt).contiguous(), v.to(self.dev, self.dt).contiguous())
        for s, t in zip(ids, toks):
            self.seqs[s].append(int(t))

    def append_attend(self, ids, toks, tol=None, rows=None):
        """One fused decode step (chunkattn_append_attend: append + attend in one
        launch), every layer in order; checked against the oracle when tol is
        given.  Returns (max abs err or None, out of the last layer)."""
        pos = [len(self.seqs[s]) for s in ids]
        k, v = self.kv(toks, pos)
        for s, t in zip(ids, toks):
            self.seqs[s].append(int(t))
        err, out = None, None
        for layer in range(self.L):
            q64 = self.queries(ids, layer)
            out = self.ca.append_attend(ids, toks if layer == 0 else None,
                                        k[:, layer].to(self.dev, self.dt).contiguous(),
                                        v[:, layer].to(self.dev, self.dt).contiguous(),
                                        q64.to(self.dev, self.dt).contiguous(), layer=layer)
            torch.cuda.synchronize()
            if tol is not None:
                ref = self.oracle(ids, q64, layer, rows=rows)
                got = out.double().cpu().numpy()
                if rows is not None:
                    got, ref = got[rows], ref[rows]
                e = float(np.abs(got - ref).max()) if got.size else 0.0
                assert np.isfinite(got).all(), "non-finite output"
                assert e <= tol, f"layer {layer}: max abs err {e} > {tol}"
                err = e if err is None else max(err, e)
        return err, out

    def queries(self, ids, layer=0):
        q = synth.q_values(self.seed, torch.as_tensor(ids), self.step, self.L, self.h, self.d, alpha=self.alpha)
        return q[:, layer].contiguous()  # [n][h][d] fp64 (exact in dtype)

    def attend(self, ids, layer=0, q64=None):
        if q64 is None:
            q64 = self.queries(ids, layer)
        out = self.ca.attend(ids, q64.to(self.dev, self.dt).contiguous(), layer=layer)
        torch.cuda.synchronize()
        return q64, out

    def oracle(self, ids, q64, layer=0, scale=None, rows=None):
        scale = scale or default_scale(self.d)
        res = np.zeros((len(ids), self.h, self.d))
        for r, sid in enumerate(ids):
            if rows is not None and r not in rows:
                continue
            toks = self.seqs[sid]
            k, v = self.kv(toks, list(range(len(toks))))
            res[r] = attend_heads_fp64(q64[r].numpy(), k[:, layer].cpu().numpy(), v[:, layer].cpu().numpy(), scale)
        return res

    def check(self, ids, tol, layer=0, rows=None):
        q64, out = self.attend(ids, layer)
        ref = self.oracle(ids, q64, layer, rows=rows)
        got = out.double().cpu().numpy()
        if rows is not None:
            got, ref = got[rows], ref[rows]
        err = float(np.abs(got - ref).max()) if got.size else 0.0
        if err > tol:  # which (row, head) cells are off
            bad = np.argwhere(np.abs(got - ref).max(axis=-1) > tol)
            print("bad (row, head):", bad[:20].tolist(), "of", got.shape[:2])
        assert np.isfinite(got).all(), "non-finite output"
        assert err <= tol, f"max abs err {err} > {tol}"
        return err, out


def build_shared(hs: Harness, n_shared, privates, seed_tag=0):
    """b sequences = shared prompt of n_shared tokens + private question of
    privates[i] tokens (seeded token ids)."""
    prompt = synth.token_ids(hs.seed, synth.TAG_SYS, seed_tag, n_shared).tolist()
    ids = []
    for i, p in enumerate(privates):
        q = synth.token_ids(hs.seed, synth.TAG_PRIV, 1000 * seed_tag + i, p).tolist()
        toks = prompt + q
        if not toks:
            toks = [1]
        ids.append(hs.add(toks)[0])
    return ids


def decode_tokens(hs: Harness, ids):
    return [int(synth.hash_py(hs.seed, synth.TAG_DECODE, s, hs.step) % 31999 + 1) for s in ids]
