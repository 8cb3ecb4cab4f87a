"""Python binding of the C ABI: `ChunkAttention` owns the torch tensors the
library computes in (K/V chunk pool, workspace) and marshals arguments.

Every step of the hot path runs in libchunkattn.so (host C++ prefix tree and
context builder, CUDA kernels).  PyTorch only provides device memory, the
current stream and process groups.  There is no CPU or eager fallback.
"""
from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np
import torch

from . import _capi as C

_DT = {torch.float32: C.CA_F32, torch.float16: C.CA_F16, torch.bfloat16: C.CA_BF16}


def _i64(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(seq, dtype=np.int64).reshape(-1))


def _i32(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(seq, dtype=np.int32).reshape(-1))


def _p64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _p32(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


class ChunkAttention:
    """Prefix-aware chunked KV cache + two-phase-partition decode attention.

    device=None builds a host-only handle (tree and tables, no kernels)."""

    def __init__(self, num_heads: int, head_dim: int, chunk_size: int, max_chunks: int, max_batch: int,
                 max_seq_len: int, dtype: torch.dtype = torch.float16, out_dtype: torch.dtype | None = None,
                 num_layers: int = 1, share_threshold: int = 2, prefix_match: bool = True, scale: float = 0.0,
                 device: str | torch.device | None = "cuda"):
        self.lib = C.lib()
        self.h, self.d, self.c, self.L = num_heads, head_dim, chunk_size, num_layers
        self.dtype = dtype
        self.out_dtype = out_dtype if out_dtype is not None else dtype
        self.device = torch.device(device) if device is not None else None
        if self.device is not None and self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        cfg = C.Config(num_heads, head_dim, chunk_size, num_layers, _DT[dtype], _DT[self.out_dtype],
                       share_threshold, 1 if prefix_match else 0, float(scale),
                       self.device.index if self.device is not None else -1, max_chunks, max_batch, max_seq_len)
        self.cfg = cfg
        ws = self.lib.chunkattn_workspace_bytes(ctypes.byref(cfg))
        if ws == 0:
            raise C.ChunkAttnError(C.CA_EINVAL, "invalid configuration")
        self.workspace_bytes = ws
        bufs = C.Buffers()
        if self.device is not None:
            shape = (num_layers, max_chunks, num_heads, chunk_size, head_dim)
            self.k_pool = torch.zeros(shape, dtype=dtype, device=self.device)
            self.v_pool = torch.zeros(shape, dtype=dtype, device=self.device)
            self.workspace = torch.zeros(ws, dtype=torch.uint8, device=self.device)
            bufs = C.Buffers(self.k_pool.data_ptr(), self.v_pool.data_ptr(), self.workspace.data_ptr(), ws)
        self._h = ctypes.c_void_p()
        C.check(self.lib.chunkattn_create(ctypes.byref(cfg), ctypes.byref(bufs), ctypes.byref(self._h)))

    # ------------------------------------------------------------------ utils
    def _stream(self):
        if self.device is None:
            return None
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _dev(self, t: torch.Tensor, shape, name: str, dtype=None):
        dtype = dtype or self.dtype
        if not (t.is_cuda and t.device == self.device):
            raise ValueError(f"{name} must be a CUDA tensor on {self.device}")
        if t.dtype != dtype:
            raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        return ctypes.c_void_p(t.data_ptr())

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self.lib.chunkattn_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------- API
    def match_prefix(self, tokens: Sequence[int]) -> int:
        t = _i32(tokens)
        m = ctypes.c_int64()
        C.check(self.lib.chunkattn_match_prefix(self._h, _p32(t), len(t), ctypes.byref(m)))
        return m.value

    def add_sequence(self, tokens: Sequence[int], k: torch.Tensor | None = None, v: torch.Tensor | None = None,
                     kv_first_pos: int = 0) -> tuple[int, int]:
        """K/V of positions kv_first_pos..n-1 as [n - kv_first_pos][L][h][d]."""
        t = _i32(tokens)
        n = len(t)
        kp = vp = None
        if self.device is not None:
            shape = (n - kv_first_pos, self.L, self.h, self.d)
            kp = self._dev(k, shape, "k")
            vp = self._dev(v, shape, "v")
        sid, m = ctypes.c_int64(), ctypes.c_int64()
        C.check(self.lib.chunkattn_add_sequence(self._h, _p32(t), n, kp, vp, kv_first_pos, self._stream(),
                                                ctypes.byref(sid), ctypes.byref(m)))
        return sid.value, m.value

    def append_kv(self, seq_ids: Sequence[int], tokens: Sequence[int], k: torch.Tensor | None = None,
                  v: torch.Tensor | None = None) -> None:
        """One decode step: k, v [n][L][h][d] in seq_ids order."""
        ids = _i64(seq_ids)
        t = _i32(tokens)
        if len(t) != len(ids):
            raise ValueError("tokens and seq_ids differ in length")
        kp = vp = None
        if self.device is not None:
            shape = (len(ids), self.L, self.h, self.d)
            kp = self._dev(k, shape, "k")
            vp = self._dev(v, shape, "v")
        C.check(self.lib.chunkattn_append_kv(self._h, len(ids), _p64(ids), _p32(t), kp, vp, self._stream()))

    def remove_sequence(self, seq_id: int) -> int:
        r = ctypes.c_int64()
        C.check(self.lib.chunkattn_remove_sequence(self._h, int(seq_id), ctypes.byref(r)))
        return r.value

    def attend(self, seq_ids: Sequence[int], q: torch.Tensor | None = None, layer: int = 0,
               out: torch.Tensor | None = None) -> torch.Tensor | None:
        """q [n][h][d] (row k = seq_ids[k]) -> out [n][h][d] in out_dtype."""
        ids = _i64(seq_ids)
        n = len(ids)
        qp = op = None
        if self.device is not None:
            qp = self._dev(q, (n, self.h, self.d), "q")
            if out is None:
                out = torch.empty((n, self.h, self.d), dtype=self.out_dtype, device=self.device)
            op = self._dev(out, (n, self.h, self.d), "out", self.out_dtype)
        C.check(self.lib.chunkattn_attend(self._h, layer, n, _p64(ids), qp, op, self._stream()))
        return out

    def append_attend(self, seq_ids: Sequence[int], tokens: Sequence[int] | None, k: torch.Tensor,
                      v: torch.Tensor, q: torch.Tensor, layer: int = 0,
                      out: torch.Tensor | None = None) -> torch.Tensor:
        """One decode step of one layer in one launch (chunkattn_append_attend):
        k, v [n][h][d] this layer's new K/V rows, q [n][h][d], all in seq_ids
        order; tokens (layer 0) the new token per sequence -> out [n][h][d]."""
        ids = _i64(seq_ids)
        n = len(ids)
        t = _i32(tokens if tokens is not None else [])
        if layer == 0 and len(t) != n:
            raise ValueError("tokens and seq_ids differ in length")
        kp = self._dev(k, (n, self.h, self.d), "k")
        vp = self._dev(v, (n, self.h, self.d), "v")
        qp = self._dev(q, (n, self.h, self.d), "q")
        if out is None:
            out = torch.empty((n, self.h, self.d), dtype=self.out_dtype, device=self.device)
        op = self._dev(out, (n, self.h, self.d), "out", self.out_dtype)
        C.check(self.lib.chunkattn_append_attend(self._h, layer, n, _p64(ids), _p32(t) if len(t) else None, kp, vp,
                                                 qp, op, self._stream()))
        return out

    def append_attend_raw(self, ids: np.ndarray, toks: np.ndarray, k_ptr: int, v_ptr: int, q_ptr: int,
                          out_ptr: int, stream_ptr: int, layer: int = 0) -> None:
        """Pre-marshalled append_attend for timing loops."""
        C.check(self.lib.chunkattn_append_attend(self._h, layer, len(ids), _p64(ids), _p32(toks),
                                                 ctypes.c_void_p(k_ptr), ctypes.c_void_p(v_ptr),
                                                 ctypes.c_void_p(q_ptr), ctypes.c_void_p(out_ptr),
                                                 ctypes.c_void_p(stream_ptr)))

    def prefill_attend(self, seq_ids: Sequence[int], first_pos: Sequence[int], q: torch.Tensor,
                       layer: int = 0, out: torch.Tensor | None = None) -> torch.Tensor:
        """Causal prefill attention of positions first_pos[k].. of each sequence
        over its whole context in the pool (chunkattn_prefill_attend): q [Q][h][d]
        packed in seq_ids order, ascending positions -> out [Q][h][d]."""
        ids = _i64(seq_ids)
        fp = _i64(first_pos)
        if len(fp) != len(ids):
            raise ValueError("first_pos and seq_ids differ in length")
        nq = q.shape[0]
        qp = self._dev(q, (nq, self.h, self.d), "q")
        if out is None:
            out = torch.empty((nq, self.h, self.d), dtype=self.out_dtype, device=self.device)
        op = self._dev(out, (nq, self.h, self.d), "out", self.out_dtype)
        C.check(self.lib.chunkattn_prefill_attend(self._h, layer, len(ids), _p64(ids), _p64(fp), qp, op,
                                                  self._stream()))
        return out

    def decode_step_host(self, ids: np.ndarray, toks: np.ndarray, in_host: torch.Tensor, out_host: torch.Tensor,
                         staging: torch.Tensor, layer: int = 0, stream_ptr: int | None = None) -> None:
        """One decode step from host buffers (chunkattn_decode_step_host): in_host
        packed [q | k_new | v_new] (pinned), out_host [n][h][d] (pinned), staging a
        device scratch tensor.  Asynchronous on the stream."""
        if in_host.is_cuda or out_host.is_cuda or not staging.is_cuda:
            raise ValueError("in_host/out_host must be host tensors and staging a device tensor")
        st = ctypes.c_void_p(stream_ptr) if stream_ptr is not None else self._stream()
        C.check(self.lib.chunkattn_decode_step_host(
            self._h, layer, len(ids), _p64(ids), _p32(toks), ctypes.c_void_p(in_host.data_ptr()),
            ctypes.c_void_p(out_host.data_ptr()), ctypes.c_void_p(staging.data_ptr()),
            staging.numel() * staging.element_size(), st))

    def attend_raw(self, layer: int, ids: np.ndarray, q_ptr: int, out_ptr: int, stream_ptr: int) -> None:
        """Pre-marshalled attend for timing loops (ids int64 contiguous)."""
        C.check(self.lib.chunkattn_attend(self._h, layer, len(ids), _p64(ids), ctypes.c_void_p(q_ptr),
                                          ctypes.c_void_p(out_ptr), ctypes.c_void_p(stream_ptr)))

    def append_raw(self, ids: np.ndarray, toks: np.ndarray, k_ptr: int, v_ptr: int, stream_ptr: int) -> None:
        C.check(self.lib.chunkattn_append_kv(self._h, len(ids), _p64(ids), _p32(toks), ctypes.c_void_p(k_ptr),
                                             ctypes.c_void_p(v_ptr), ctypes.c_void_p(stream_ptr)))

    def batch_order(self) -> list[int]:
        cap = 1 << 20
        buf = np.zeros(cap, dtype=np.int64)
        n = ctypes.c_int64()
        C.check(self.lib.chunkattn_batch_order(self._h, _p64(buf), cap, ctypes.byref(n)))
        return buf[:n.value].tolist()

    def export_context(self) -> str:
        ln = ctypes.c_size_t()
        self.lib.chunkattn_export_context(self._h, None, 0, ctypes.byref(ln))
        buf = ctypes.create_string_buffer(ln.value + 1)
        C.check(self.lib.chunkattn_export_context(self._h, buf, ln.value + 1, ctypes.byref(ln)))
        return buf.value.decode()

    def memory_stats(self) -> dict:
        a = (ctypes.c_int64 * 6)()
        C.check(self.lib.chunkattn_memory_stats(self._h, a))
        return dict(zip(["used", "free", "created", "hwm", "kv_bytes", "waste_slots"], list(a)))

    def counters(self) -> dict:
        a = (ctypes.c_int64 * 6)()
        C.check(self.lib.chunkattn_counters(self._h, a))
        return dict(zip(["builds", "uploads", "upload_bytes", "launches", "epoch", "slots"], list(a)))

    def schedule_info(self) -> dict:
        a = (ctypes.c_int64 * 9)()
        C.check(self.lib.chunkattn_schedule_info(self._h, a))
        return dict(zip(["dk", "dk_cs", "dk_groups", "dk_blocks", "dk_units", "dk_hg", "fused", "sf_ctas", "dk_um"],
                        list(a)))

    def set_option(self, key: str, value: int) -> None:
        C.check(self.lib.chunkattn_set_option(self._h, key.encode(), int(value)))

    def kernel_times(self) -> dict:
        """{kind: (total ms, launches)} since the last call (option "kernel_events")."""
        ms = (ctypes.c_double * 4)()
        n = (ctypes.c_int64 * 4)()
        C.check(self.lib.chunkattn_kernel_times(self._h, ms, n))
        return {k: (ms[i], n[i]) for i, k in enumerate(["append", "chunk_first", "seq_first", "copy"])}

    def download_tables(self) -> np.ndarray:
        ln = ctypes.c_size_t()
        self.lib.chunkattn_download_tables(self._h, None, 0, ctypes.byref(ln), self._stream())
        buf = np.zeros(max(1, ln.value // 4), dtype=np.int32)
        C.check(self.lib.chunkattn_download_tables(self._h, buf.ctypes.data_as(ctypes.c_void_p), ln.value,
                                                   ctypes.byref(ln), self._stream()))
        return buf[:ln.value // 4]

    def host_tables(self) -> np.ndarray:
        """The host-built context tables (int32) of the current epoch."""
        ln = ctypes.c_size_t()
        self.lib.chunkattn_host_tables(self._h, None, 0, ctypes.byref(ln))
        buf = np.zeros(max(1, ln.value // 4), dtype=np.int32)
        C.check(self.lib.chunkattn_host_tables(self._h, buf.ctypes.data_as(ctypes.c_void_p), ln.value,
                                               ctypes.byref(ln)))
        return buf[:ln.value // 4]
