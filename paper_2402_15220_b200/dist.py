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
permuted to [n][h][d].  RowShardedChunkAttention splits the sequences of one
batch instead (contiguous rows make row slices cheap); shared
chunks straddling a cut are replicated on the ranks that use them.
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


def _all_gather_stacked(x: torch.Tensor, group=None) -> torch.Tensor:
    """[...] on every rank -> [W][...] on every rank: one NCCL
    all_gather_into_tensor for CUDA tensors on an NCCL group, else (gloo: CPU
    tests, or several ranks sharing one GPU in tests) a list all-gather staged
    through host memory."""
    world = dist.get_world_size(group)
    if x.is_cuda and dist.get_backend(group) == "nccl":
        buf = torch.empty((world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(buf, x.contiguous(), group=group)
        return buf
    xc = x.detach().contiguous().cpu()
    parts = [torch.empty_like(xc) for _ in range(world)]
    dist.all_gather(parts, xc, group=group)
    return torch.stack(parts).to(x.device)


def gather_heads(out_local: torch.Tensor, group=None) -> torch.Tensor:
    """[n][h_local][d] on every rank -> [n][W * h_local][d] (rank-major heads)."""
    world = dist.get_world_size(group)
    if world == 1:
        return out_local
    n, hl, d = out_local.shape
    buf = _all_gather_stacked(out_local, group)
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

    def append_attend_local(self, seq_ids, tokens, k, v, q, layer=0):
        """One fused decode step on this rank's heads: k, v, q [n][h][d] (all
        heads) -> this rank's output slice [n][h/W][d]."""
        return self.ca.append_attend(seq_ids, tokens, self._heads(k), self._heads(v), self._heads(q), layer=layer)

    def append_attend(self, seq_ids, tokens, k, v, q, layer=0):
        """One fused decode step -> [n][h][d] on every rank (one all-gather)."""
        return gather_heads(self.append_attend_local(seq_ids, tokens, k, v, q, layer), self.group)

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
        parts = _all_gather_stacked(mine, self.group)
        return all(torch.equal(p, parts[0]) for p in parts)


class RowShardedChunkAttention:
    """The sequence (row) split of one batch (large batches): rank
    r holds the sequences assigned to it, with all their heads.  Sequences
    whose first chunk carries the same tokens (one shared prefix, one run of
    the forest) go to the same rank -- cuts fall between runs where the load
    allows, and a shared chunk whose sequences do land on several ranks is
    simply held by each of them (replicated straddling chunk).  Every rank
    replays the full op stream for the assignment (deterministic) but adds,
    appends and removes only its own sequences; attend computes the local rows
    and one all-gather (rows padded to the largest rank) reassembles the
    caller's order.  Tree and tables are per rank: the (C, i, j) of a rank are
    the global ones clipped to its rows."""

    def __init__(self, num_heads: int, head_dim: int, chunk_size: int, max_chunks: int, max_batch: int,
                 max_seq_len: int, group=None, device=None, **kw):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.h, self.d, self.c = num_heads, head_dim, chunk_size
        self.ca = ChunkAttention(num_heads, head_dim, chunk_size, max_chunks, max_batch, max_seq_len,
                                 device=device, **kw)
        self.owner = {}     # global sequence id -> rank
        self.local = {}     # global id -> this rank's library id
        self.group_rank = {}  # first-chunk tokens -> rank
        self.load = [0] * self.world
        self.next_id = 0

    def _assign(self, tokens) -> int:
        key = tuple(tokens[:self.c]) if len(tokens) >= self.c else None
        fair = (sum(self.load) + 1 + self.world - 1) // self.world
        r = self.group_rank.get(key) if key is not None else None
        if r is None or self.load[r] >= fair + 1:  # a new run, or its rank is over its share
            r = min(range(self.world), key=lambda x: (self.load[x], x))
            if key is not None and key not in self.group_rank:
                self.group_rank[key] = r
        return r

    def add_sequence(self, tokens, k=None, v=None, kv_first_pos=0):
        """Every rank calls this with the same tokens (k / v may be None on
        ranks that do not own the sequence).  Returns the global id."""
        gid = self.next_id
        self.next_id += 1
        r = self._assign(list(tokens))
        self.owner[gid] = r
        self.load[r] += 1
        if r == self.rank:
            lid, _ = self.ca.add_sequence(tokens, k, v, kv_first_pos)
            self.local[gid] = lid
        return gid

    def remove_sequence(self, gid):
        r = self.owner.pop(gid)
        self.load[r] -= 1
        if r == self.rank:
            self.ca.remove_sequence(self.local.pop(gid))

    def _mine(self, seq_ids):
        return [i for i, g in enumerate(seq_ids) if self.owner[g] == self.rank]

    def append_attend(self, seq_ids, tokens, k, v, q, layer=0):
        """One decode step for all live sequences: k, v, q [n][h][d] in seq_ids
        order -> out [n][h][d] (one all-gather)."""
        mine = self._mine(seq_ids)
        n = len(seq_ids)
        counts = [sum(1 for g in seq_ids if self.owner[g] == r) for r in range(self.world)]
        width = max(counts) if counts else 0
        part = torch.zeros((width, self.h, self.d), dtype=self.ca.out_dtype, device=q.device)
        if mine:
            idx = torch.tensor(mine, device=q.device)
            out = self.ca.append_attend([self.local[seq_ids[i]] for i in mine],
                                        [tokens[i] for i in mine] if tokens is not None else None,
                                        k[idx].contiguous(), v[idx].contiguous(), q[idx].contiguous(), layer=layer)
            part[:len(mine)] = out
        parts = _all_gather_stacked(part, self.group) if self.world > 1 else part[None]
        full = torch.empty((n, self.h, self.d), dtype=part.dtype, device=q.device)
        for r in range(self.world):
            rows = [i for i, g in enumerate(seq_ids) if self.owner[g] == r]
            if rows:
                full[torch.tensor(rows, device=q.device)] = parts[r, :len(rows)]
        return full
