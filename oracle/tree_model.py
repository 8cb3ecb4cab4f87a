"""Prefix-tree replay oracle (C3) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's oracle legs may import this
module.  It shares no code with the C++ host library; it replays the same op
stream with plain Python dicts and lists and emits the canonical tables that
the C++ `chunkattn_export_context` must reproduce byte for byte.

Follows PAPER.md §3.1 (PAKV, lines 505-513):
  * "Each node defines a chunk C storing ... c context tokens ... key ...
    value" (:505); "Each path in the prefix tree defines a sequence" (:505);
    "Multiple trees (a forest)" (:505).
  * three scenarios (:507): "new sequence joins" -> add_sequence (search and
    insert a path), "completed sequence leaves" -> remove_sequence (delete its
    path), "all sequences decode one token" -> append ("append new tokens into
    leaf chunks or grow a new chunk when the leaf chunk is full").
  * pool allocator (:509): "returns a chunk from the free list or allocates
    fresh memory"; chunks are "returned to the allocator once a sequence is
    completed" and never released to the OS.
  * contiguity (:513): "sequences covered by each chunk ... are contiguous in
    the sequence index dimension" — produced by the DFS row order below.
and the context of PAPER.md:162 (§3.3): (C, i, j) tuples plus per-sequence
private chunk lists.

Readings (DESIGN.md ledger): T1 only full aligned chunks are matched/shared;
T2 LIFO free list over a bump pointer, release leaf->root, acquire in path /
call order; T3' siblings (and forest roots) ordered by chunk creation serial,
sequences terminating at a node come before its children, ordered by seq id;
T4 epoch bumps on any acquire/release/add/remove; T5 canonical export format.

Pins (tests/test_oracle_tree.py): the paper's Fig-2 worked example
 reproduced exactly, chunk arithmetic from SPEC.md:78/88/126,
structural invariants after every fuzz op, and the order-free sharing
definition in oracle/sharing.py.
"""
from __future__ import annotations


class PoolExhausted(Exception):
    pass


class _Chunk:
    __slots__ = ("id", "serial", "parent", "children", "start_pos", "tokens", "ref", "terms")

    def __init__(self, cid, serial, parent, start_pos):
        self.id = cid
        self.serial = serial
        self.parent = parent          # _Chunk or None (root)
        self.children = []            # creation-serial order (T3')
        self.start_pos = start_pos
        self.tokens = []
        self.ref = 0
        self.terms = set()            # seq ids whose path ends here


class TreeModel:
    def __init__(self, chunk_size, max_chunks, share_threshold=2, prefix_match=True):
        self.c = chunk_size
        self.max_chunks = max_chunks
        self.share_threshold = share_threshold
        self.prefix_match = prefix_match
        self.roots = []
        self.chunks = {}              # id -> _Chunk (live)
        self.free = []                # LIFO stack of released ids
        self.created = 0
        self.hwm = 0
        self.serial = 0
        self.seqs = {}                # seq id -> list of _Chunk (path)
        self.seq_len = {}
        self.next_seq = 0
        self.epoch = 0

    # ------------------------------------------------------------ pool ----
    def _available(self):
        return len(self.free) + (self.max_chunks - self.created)

    def _acquire(self, parent, start_pos):
        if self.free:
            cid = self.free.pop()
        elif self.created < self.max_chunks:
            cid = self.created
            self.created += 1
        else:
            raise PoolExhausted()
        ch = _Chunk(cid, self.serial, parent, start_pos)
        self.serial += 1
        self.chunks[cid] = ch
        (parent.children if parent is not None else self.roots).append(ch)
        self.hwm = max(self.hwm, len(self.chunks))
        return ch

    def _release(self, ch):
        sib = ch.parent.children if ch.parent is not None else self.roots
        sib.remove(ch)
        del self.chunks[ch.id]
        self.free.append(ch.id)

    # ------------------------------------------------------------ ops -----
    def _match(self, tokens):
        """Matched chunks along the path (T1: full, aligned, equal tuples)."""
        c = self.c
        path = []
        if not self.prefix_match:
            return path
        cands = self.roots
        k = 0
        while (k + 1) * c <= len(tokens):
            tup = list(tokens[k * c:(k + 1) * c])
            hit = None
            for ch in cands:
                if len(ch.tokens) == c and ch.tokens == tup:
                    hit = ch
                    break
            if hit is None:
                break
            path.append(hit)
            cands = hit.children
            k += 1
        return path

    def match_prefix(self, tokens):
        return len(self._match(tokens)) * self.c

    def add_sequence(self, tokens):
        """Insert a path; returns (seq_id, matched_tokens, new chunk ids in path order)."""
        tokens = [int(t) for t in tokens]
        if len(tokens) == 0:
            raise ValueError("empty sequence")
        c = self.c
        path = self._match(tokens)
        matched = len(path) * c
        need = -(-(len(tokens) - matched) // c)
        if need > self._available():
            raise PoolExhausted()
        parent = path[-1] if path else None
        new = []
        for k in range(need):
            start = matched + k * c
            ch = self._acquire(parent, start)
            ch.tokens = tokens[start:start + c]
            new.append(ch)
            parent = ch
        sid = self.next_seq
        self.next_seq += 1
        full = path + new
        for ch in full:
            ch.ref += 1
        full[-1].terms.add(sid)
        self.seqs[sid] = full
        self.seq_len[sid] = len(tokens)
        self.epoch += 1
        return sid, matched, [ch.id for ch in new]

    def append(self, seq_ids, tokens):
        """One decode step for several sequences, processed in call order.

        Returns [(chunk id, slot, structural)] per sequence."""
        seq_ids = [int(s) for s in seq_ids]
        for s in seq_ids:
            if s not in self.seqs:
                raise KeyError(s)
        if len(set(seq_ids)) != len(seq_ids):
            raise ValueError("duplicate seq id")
        need = 0
        for s in seq_ids:
            last = self.seqs[s][-1]
            if not (last.ref == 1 and len(last.tokens) < self.c):
                need += 1
        if need > self._available():
            raise PoolExhausted()
        out = []
        for s, t in zip(seq_ids, tokens):
            path = self.seqs[s]
            last = path[-1]
            if last.ref == 1 and len(last.tokens) < self.c:
                slot = len(last.tokens)
                last.tokens.append(int(t))
                out.append((last.id, slot, False))
            else:
                ch = self._acquire(last, self.seq_len[s])
                ch.tokens = [int(t)]
                ch.ref = 1
                last.terms.discard(s)
                ch.terms.add(s)
                path.append(ch)
                out.append((ch.id, 0, True))
                self.epoch += 1
            self.seq_len[s] += 1
        return out

    def remove_sequence(self, sid):
        """Delete a path; returns the released chunk ids (leaf -> root order)."""
        path = self.seqs.pop(sid)
        del self.seq_len[sid]
        path[-1].terms.discard(sid)
        released = []
        for ch in reversed(path):
            ch.ref -= 1
            if ch.ref == 0:
                self._release(ch)
                released.append(ch.id)
        self.epoch += 1
        return released

    # ------------------------------------------------------------ context --
    def _dfs(self):
        """Pre-order chunk list with row ranges; rows assigned per T3'."""
        order = []            # seq ids by row
        recs = []             # (chunk, i, j) pre-order

        def visit(ch):
            idx = len(recs)
            recs.append(None)
            i = len(order)
            order.extend(sorted(ch.terms))
            for kid in ch.children:
                visit(kid)
            recs[idx] = (ch, i, len(order) - 1)

        for r in self.roots:
            visit(r)
        return order, recs

    def batch_order(self):
        return self._dfs()[0]

    def context(self):
        order, recs = self._dfs()
        row_of = {s: r for r, s in enumerate(order)}
        thr = self.share_threshold
        shared = [(ch.id, i, j) for (ch, i, j) in recs if ch.ref >= thr]
        private = [[ch.id for ch in self.seqs[s] if ch.ref < thr] for s in order]
        return {
            "order": order,
            "row_of": row_of,
            "chunks": [(ch.id, ch.parent.id if ch.parent else -1, ch.start_pos,
                        len(ch.tokens), ch.ref, ch.tokens[0], ch.tokens[-1], i, j)
                       for (ch, i, j) in recs],
            "shared": shared,
            "private": private,
            "tuples": [(ch.id, i, j) for (ch, i, j) in recs],
            "alloc": (len(self.chunks), len(self.free), self.created, self.hwm),
        }

    def export(self):
        """Canonical text (T5); must equal chunkattn_export_context byte for byte."""
        ctx = self.context()
        lines = ["chunks:"]
        for (cid, par, sp, ln, ref, ft, lt, i, j) in ctx["chunks"]:
            lines.append(f"{cid} {par} {sp} {ln} {ref} {ft} {lt}")
        lines.append("order:" + "".join(f" {s}" for s in ctx["order"]))
        lines.append("shared:" + "".join(f" ({c},{i},{j})" for (c, i, j) in ctx["shared"]))
        for r, lst in enumerate(ctx["private"]):
            lines.append(f"private[{r}]:" + "".join(f" {c}" for c in lst))
        lines.append("tuples:" + "".join(f" ({c},{i},{j})" for (c, i, j) in ctx["tuples"]))
        u, f, cr, hw = ctx["alloc"]
        lines.append(f"alloc: {u} {f} {cr} {hw}")
        return "\n".join(lines) + "\n"

    def memory_stats(self):
        """(used, free, created, hwm, waste_slots): waste = unused aligned slots."""
        waste = sum(self.c - len(ch.tokens) for ch in self.chunks.values())
        return (len(self.chunks), len(self.free), self.created, self.hwm, waste)

    # ------------------------------------------------------------ helpers --
    def path_ids(self, sid):
        return [ch.id for ch in self.seqs[sid]]

    def tokens_of(self, sid):
        out = []
        for ch in self.seqs[sid]:
            out.extend(ch.tokens)
        return out

    def token_slots(self, sid):
        """(chunk id, slot) of every token of the sequence, position order."""
        out = []
        for ch in self.seqs[sid]:
            for k in range(len(ch.tokens)):
                out.append((ch.id, k))
        return out
