"""Multi-GPU partitioning of decode attention.

Attention heads are independent ("the head dimension is always partitioned",
PAPER.md:66 §3.2), so W ranks split the h heads: rank r owns heads
[r h/W, (r+1) h/W) and holds only their K/V in its chunk pool.  The prefix tree
and the context tables are head-independent: every rank replays the same host
op stream (add / append / remove) and, the library being deterministic (tree
rules T1-T3', fixed schedule), builds bit-identical trees -- checked by
`tables_consistent()` without any per-step collective.  Both phases run
rank-locally; the only data-path exchange is one all-gather of the per-rank
outputs [n][h/W][d] (NCCL over NVLink on GPUs, gloo on CPU for tests),
permuted to [n][h][d].  Independent batches per rank (the bench's weak
scaling) need no collective at all.
"""
from __future__ import annotations

import hashlib

import torch
import torch.distributed as dist

from .attention import ChunkAttention


def head_range(num_heads: int, world: int, rank: int) -> tuple[int, int]:
    if num_heads % world:
        raise ValueError(f"{num_heads} heads do not split over {world} ranks")
    per = num_heads // world
    return rank * per, (rank + 1) * per


def gather_heads(out_local: torch.Tensor, group=None) -> torch.Tensor:
    """[n][h_local][d] on every rank -> [n][W * h_local][d] (rank-major heads)."""
    world = dist.get_world_size(group)
    if world == 1:
        return out_local
    n, hl, d = out_local.shape
    if out_local.is_cuda:
        buf = torch.empty((world, n, hl, d), dtype=out_local.dtype, device=out_local.device)
        dist.all_gather_into_tensor(buf, out_local.contiguous(), group=group)
    else:  # gloo: list all-gather
        parts = [torch.empty_like(out_local) for _ in range(world)]
        dist.all_gather(parts, out_local.contiguous(), group=group)
        buf = torch.stack(parts)
    return buf.permute(1, 0, 2, 3).reshape(n, world * hl, d)


class ShardedChunkAttention:
    """ChunkAttention over the heads of this rank; same API with full-head tensors."""

    def __init__(self, num_heads: int, head_dim: int, chunk_size: int, max_chunks: int, max_batch: int,
                 max_seq_len: int, group=None, device=None, **kw):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.h = num_heads
        self.h0, self.h1 = head_range(num_heads, self.world, self.rank)
        self.ca = ChunkAttention(self.h1 - self.h0, head_dim, chunk_size, max_chunks, max_batch, max_seq_len,
                                 device=device, **kw)

    def _heads(self, x):  # [..., h, d] -> this rank's slice, contiguous
        return None if x is None else x[..., self.h0:self.h1, :].contiguous()

    def match_prefix(self, tokens):
        return self.ca.match_prefix(tokens)

    def add_sequence(self, tokens, k=None, v=None, kv_first_pos=0):
        """k, v: [n - kv_first_pos][L][h][d] (all heads); this rank keeps its slice."""
        return self.ca.add_sequence(tokens, self._heads(k), self._heads(v), kv_first_pos)

    def append_kv(self, seq_ids, tokens, k=None, v=None):
        return self.ca.append_kv(seq_ids, tokens, self._heads(k), self._heads(v))

    def remove_sequence(self, seq_id):
        return self.ca.remove_sequence(seq_id)

    def attend_local(self, seq_ids, q, layer=0):
        """q [n][h][d] -> this rank's output slice [n][h/W][d]."""
        return self.ca.attend(seq_ids, self._heads(q), layer=layer)

    def attend(self, seq_ids, q, layer=0):
        """q [n][h][d] -> [n][h][d] on every rank (one all-gather)."""
        return gather_heads(self.attend_local(seq_ids, q, layer), self.group)

    def tables_digest(self) -> bytes:
        return hashlib.sha256(self.ca.export_context().encode()).digest()

    def tables_consistent(self) -> bool:
        """All ranks hold byte-identical prefix trees / contexts."""
        if self.world == 1:
            return True
        mine = torch.tensor(list(self.tables_digest()), dtype=torch.uint8)
        if dist.get_backend(self.group) == "nccl":
            mine = mine.cuda()
        parts = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(parts, mine, group=self.group)
        return all(torch.equal(p, parts[0]) for p in parts)
