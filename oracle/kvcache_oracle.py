"""TEST INFRASTRUCTURE ONLY — pure-Python restatement of the reference paged
KV cache (/root/reference/proj/core/src/kv_cache.cc, radix_tree.cc,
kv_addr.cc), the checker for the B200 library's bookkeeping and page
contents.  The toy-model arithmetic comes from the C restatement
(oracle/hashmodel.c).  Pinned against the compiled reference
(oracle/_ref/libmicrokv_ref.so) by tests/test_oracle_pinning.py.

Method names and error behaviour match paper_2412_12488_b200.KVCache (and
the reference class), so one scenario script can drive all three.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it.
Sizes: meant for the tiny config and small 8B-shape cases (pages are a
numpy array in the reference's [page][slot][layer][word] layout).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import hashmodel as hm

try:  # share the error/enum types with the product mirror when importable
    from paper_2412_12488_b200.kvcache import (ApplyStatus, ErrorCode, FillState, KVAddrInfo,
                                               PrepRecvResult, SequenceRecordInfo,
                                               SplitserveError)
except Exception:  # pragma: no cover - the package is always present in this repo
    raise


def _err(code: ErrorCode, detail: str) -> SplitserveError:
    return SplitserveError(int(code) + 1, f"{code.name}: {detail}")


# ---------------------------------------------------------------------------
# RadixTree (radix_tree.cc)
# ---------------------------------------------------------------------------
class _Node:
    __slots__ = ("edge", "kids", "ref", "lru", "pinned")

    def __init__(self, edge=(), ref=-1, lru=0, pinned=False):
        self.edge = list(edge)
        self.kids: dict = {}
        self.ref = ref
        self.lru = lru
        self.pinned = pinned


class RadixTree:
    def __init__(self):
        self.root = _Node()
        self.clock = 0
        self.touch: dict = {}

    def _touch(self, seq):  # radix_tree.cc:24-26
        if seq >= 0:
            self.clock += 1
            self.touch[seq] = self.clock

    @staticmethod
    def _common(node, tokens, pos):
        c = 0
        while c < len(node.edge) and pos + c < len(tokens) and node.edge[c] == tokens[pos + c]:
            c += 1
        return c

    def MatchPrefix(self, tokens):  # radix_tree.cc:28-53
        tokens = list(tokens)
        match_len, seq = 0, -1
        node, pos = self.root, 0
        self.clock += 1
        while pos < len(tokens):
            child = node.kids.get(tokens[pos])
            if child is None:
                break
            c = self._common(child, tokens, pos)
            if c > 0:
                child.lru = self.clock
                match_len, seq = pos + c, child.ref
            if c < len(child.edge):
                break
            pos += c
            node = child
        self._touch(seq)
        return match_len, seq

    def Insert(self, tokens, seq):  # radix_tree.cc:55-94
        tokens = list(tokens)
        node, pos = self.root, 0
        self.clock += 1
        while pos < len(tokens):
            child = node.kids.get(tokens[pos])
            if child is None:
                node.kids[tokens[pos]] = _Node(tokens[pos:], seq, self.clock)
                self._touch(seq)
                return
            c = self._common(child, tokens, pos)
            if c < len(child.edge):
                tail = _Node(child.edge[c:], child.ref, child.lru, child.pinned)
                tail.kids = child.kids
                child.edge = child.edge[:c]
                child.kids = {tail.edge[0]: tail}
            child.ref = seq
            child.lru = self.clock
            pos += c
            node = child
        self._touch(seq)

    def Remove(self, seq):  # radix_tree.cc:96-124
        def visit(node):
            for tok in sorted(node.kids):
                if not visit(node.kids[tok]):
                    del node.kids[tok]
            if node.ref == seq:
                if not node.kids:
                    return False
                node.ref = node.kids[min(node.kids)].ref
            return True

        for tok in sorted(self.root.kids):
            if not visit(self.root.kids[tok]):
                del self.root.kids[tok]
        self.touch.pop(seq, None)

    def Pin(self, prefix, flag):  # radix_tree.cc:126-143
        prefix = list(prefix)
        node, pos = self.root, 0
        while pos < len(prefix):
            child = node.kids.get(prefix[pos])
            if child is None:
                return
            c = self._common(child, prefix, pos)
            if c > 0:
                child.pinned = flag
            if c < len(child.edge):
                return
            pos += c
            node = child

    def HasPinnedNode(self, seq):  # radix_tree.cc:145-157
        stack = [self.root]
        while stack:
            n = stack.pop()
            if n.ref == seq and n.pinned:
                return True
            stack.extend(n.kids.values())
        return False

    def Contains(self, seq):
        return seq in self.touch

    def LastTouch(self, seq):
        return self.touch.get(seq, 0)

    def SequencesByLru(self):  # radix_tree.cc:166-175
        return [s for (t, s) in sorted((t, s) for s, t in self.touch.items())]

    def NodeCount(self):
        n, stack = 0, list(self.root.kids.values())
        while stack:
            x = stack.pop()
            n += 1
            stack.extend(x.kids.values())
        return n


# ---------------------------------------------------------------------------
# KVAddrInfo helpers (kv_addr.cc:16-51)
# ---------------------------------------------------------------------------
def addr_validate(a: KVAddrInfo):
    seen, total = set(), 0
    for (p, b, c) in a.ranges:
        if not (c > 0 and b >= 0):
            raise _err(ErrorCode.InvalidArgument, "bad slot range")
        for s in range(c):
            if (p, b + s) in seen:
                raise _err(ErrorCode.InvalidArgument, "overlapping slot ranges")
            seen.add((p, b + s))
        total += c
    if total != a.token_count:
        raise _err(ErrorCode.AddrMismatch, "slot counts do not cover token_count")


def addr_slice(a: KVAddrInfo, begin, end) -> KVAddrInfo:
    if not (begin >= a.token_begin and end <= a.token_begin + a.token_count and begin <= end):
        raise _err(ErrorCode.InvalidArgument, "slice outside address")
    ranges, pos = [], a.token_begin
    for (p, b, c) in a.ranges:
        lo, hi = max(pos, begin), min(pos + c, end)
        if lo < hi:
            ranges.append((p, b + (lo - pos), hi - lo))
        pos += c
    return KVAddrInfo(ranges, begin, end - begin)


# ---------------------------------------------------------------------------
# KVCache (kv_cache.cc)
# ---------------------------------------------------------------------------
@dataclass
class _Window:
    range: tuple
    expected: int
    received: int = 0
    complete: bool = False
    applied: set = field(default_factory=set)


@dataclass
class _Record:
    id: int
    tokens: list
    parent: int = -1
    fork_len: int = 0
    refcount: int = 0
    own_pages: list = field(default_factory=list)
    alloc_len: int = 0
    committed_hint: int = 0
    finished: bool = False
    fold_frontier: int = 0
    fold_sums: list = field(default_factory=list)
    prefix_digest: int = 0
    digest_len: int = 0
    window: Optional[_Window] = None


class _Plan:
    def __init__(self):
        self.entries: list = []
        self.sends: list = []
        self.next_layer = 0
        self.total_outputs = 0


def resolve_end_index(n, end):  # kv_cache.cc:13-18
    e = n + end if end < 0 else end
    if end == 0:
        raise _err(ErrorCode.InvalidArgument, "end = 0 is invalid")
    if not (0 < e <= n):
        raise _err(ErrorCode.InvalidArgument, "end out of range")
    return e


M64 = (1 << 64) - 1


class KVCache:
    impl = "python-restatement"

    def __init__(self, num_pages=4096, page_size=16, layers=4, dim=8, vocab=256,
                 hash_seed=hm.DEFAULT_HASH_SEED, device=None, rank=0, lib=None):
        if num_pages < 1:
            raise _err(ErrorCode.InvalidArgument, "num_pages must be >= 1")
        if page_size < 1 or page_size & (page_size - 1):
            raise _err(ErrorCode.InvalidArgument, "page_size must be a power of two")
        self.num_pages, self.page_size, self.layers, self.dim = num_pages, page_size, layers, dim
        self.vocab, self.hash_seed, self.rank = vocab, hash_seed, rank
        P, L, W = page_size, layers, dim
        self.values = np.zeros((num_pages, P, L, W), dtype=np.uint64)  # kv_cache.cc:37
        self.fill = np.zeros((num_pages, P, L), dtype=np.uint8)
        self.expecting = np.zeros((num_pages, P), dtype=np.uint8)
        self.owner = [-1] * num_pages
        self.free_pages = list(range(num_pages - 1, -1, -1))  # kv_cache.cc:45-46
        self.records: dict = {}
        self.pending: list = []
        self.tree = RadixTree()
        self.completed: list = []

    # -- helpers --------------------------------------------------------------
    def _get(self, seq) -> _Record:
        if seq not in self.records:
            raise _err(ErrorCode.UnknownSequence, f"sequence {seq}")
        return self.records[seq]

    def _resolve(self, rec, pos):  # kv_cache.cc:67-77
        r = rec
        while pos < r.fork_len:
            r = self._get(r.parent)
        idx = pos - r.fork_len
        if not idx < len(r.own_pages) * self.page_size:
            raise _err(ErrorCode.Internal, "position not allocated")
        return r.own_pages[idx // self.page_size], idx % self.page_size

    def _pages_needed(self, rec, upto):  # kv_cache.cc:79-84
        idx = upto - rec.fork_len
        if idx <= 0:
            return 0
        return max(0, (idx + self.page_size - 1) // self.page_size - len(rec.own_pages))

    def _advance_committed(self, rec):  # kv_cache.cc:86-102
        pos = max(rec.committed_hint, rec.fork_len)
        while pos < rec.alloc_len and pos < len(rec.tokens):
            pg, sl = self._resolve(rec, pos)
            if (self.fill[pg, sl] == 0).any():
                break
            pos += 1
        rec.committed_hint = max(rec.committed_hint, pos)

    def _touch_lru(self, rec):  # kv_cache.cc:104-110
        if self.tree.Contains(rec.id):
            n = min(rec.committed_hint, len(rec.tokens))
            if n > 0:
                self.tree.Insert(rec.tokens[:n], rec.id)

    # -- hash model scalars -------------------------------------------------------
    def InitialPrefixDigest(self):
        return hm.initial_prefix_digest(self.hash_seed)

    def Embed(self, token, pos):
        return hm.embed(token, pos, self.hash_seed)

    def SampleToken(self, h):
        return hm.sample_token(h, self.vocab)

    # -- declaration stage ----------------------------------------------------------
    def MatchPrefixSeq(self, tokens):  # kv_cache.cc:112-118
        return self.tree.MatchPrefix(tokens)

    def MatchPrefix(self, tokens):
        return self.tree.MatchPrefix(tokens)[0]

    def CreateSequence(self, seq, tokens):  # kv_cache.cc:120-131
        if seq in self.records:
            raise _err(ErrorCode.DuplicateSequence, f"sequence {seq}")
        self.records[seq] = _Record(seq, list(tokens), fold_sums=[0] * self.layers,
                                    prefix_digest=self.InitialPrefixDigest())

    def ForkSequence(self, parent, child, fork_len, child_tokens=()):  # kv_cache.cc:133-166
        p = self._get(parent)
        if child in self.records:
            raise _err(ErrorCode.DuplicateSequence, f"sequence {child}")
        self._advance_committed(p)
        if fork_len > p.committed_hint:
            raise _err(ErrorCode.ForkBeyondCommitted,
                       f"fork_len {fork_len} > committed {p.committed_hint}")
        child_tokens = list(child_tokens)
        if not child_tokens:
            child_tokens = p.tokens[:fork_len]
        else:
            if len(child_tokens) < fork_len:
                raise _err(ErrorCode.InvalidArgument, "child tokens shorter than fork_len")
            if child_tokens[:fork_len] != p.tokens[:fork_len]:
                raise _err(ErrorCode.InvalidArgument, "child tokens diverge inside the fork prefix")
        rec = _Record(child, child_tokens, parent=parent if fork_len > 0 else -1,
                      fork_len=fork_len, alloc_len=fork_len, committed_hint=fork_len,
                      fold_sums=[0] * self.layers, prefix_digest=self.InitialPrefixDigest())
        if rec.parent >= 0:
            p.refcount += 1
        self.records[child] = rec
        self._touch_lru(p)

    def EnsureAllocated(self, seq, upto):  # kv_cache.cc:168-183
        rec = self._get(seq)
        if upto > len(rec.tokens):
            raise _err(ErrorCode.InvalidArgument, "allocation beyond known tokens")
        need = self._pages_needed(rec, upto)
        if need > len(self.free_pages):
            raise _err(ErrorCode.OutOfPages, f"{need} pages needed, {len(self.free_pages)} free")
        for _ in range(need):
            pg = self.free_pages.pop()
            self.owner[pg] = seq
            rec.own_pages.append(pg)
        rec.alloc_len = rec.fork_len + len(rec.own_pages) * self.page_size

    def AppendToken(self, seq, t):  # kv_cache.cc:185
        self._get(seq).tokens.append(int(t))

    def PrepRecv(self, seq, tokens, end):  # kv_cache.cc:187-229
        tokens = list(tokens)
        if not tokens:
            raise _err(ErrorCode.InvalidArgument, "empty prompt")
        if seq in self.records:
            raise _err(ErrorCode.DuplicateSequence, f"sequence {seq}")
        e = resolve_end_index(len(tokens), end)
        m, mseq = self.tree.MatchPrefix(tokens[:e])
        need = (e - m + self.page_size - 1) // self.page_size
        if need > len(self.free_pages):
            raise _err(ErrorCode.OutOfPages, f"{need} pages needed, {len(self.free_pages)} free")
        if m > 0:
            self.ForkSequence(mseq, seq, m, tokens)
        else:
            self.CreateSequence(seq, tokens)
        self.EnsureAllocated(seq, e)
        addr = self.BuildAddr(seq, (m, e))
        rec = self.records[seq]
        for pos in range(m, e):
            pg, sl = self._resolve(rec, pos)
            self.expecting[pg, sl] = 1
        if e > m:
            rec.window = _Window((m, e), (e - m) * self.layers)
        return PrepRecvResult(m, addr)

    def MarkSend(self, seq, token_range, dest, dest_addr, user_tag=0):  # kv_cache.cc:231-243
        rec = self._get(seq)
        b, e = token_range
        if not (b >= 0 and e <= len(rec.tokens) and b <= e):
            raise _err(ErrorCode.InvalidArgument, "send range outside sequence")
        if dest_addr.token_count != e - b:
            raise _err(ErrorCode.AddrMismatch, f"destination covers {dest_addr.token_count} "
                                               f"tokens, range has {e - b}")
        if dest_addr.token_begin != b:
            raise _err(ErrorCode.AddrMismatch, "destination token_begin mismatch")
        self.pending.append((seq, (b, e), dest, dest_addr, user_tag))

    def BeginForward(self, batch):  # kv_cache.cc:245-306
        plan, seen = _Plan(), set()
        for ent in batch:
            rec = self._get(ent.seq)
            if ent.seq in seen:
                raise _err(ErrorCode.Internal, "sequence batched twice")
            seen.add(ent.seq)
            b, e = ent.range
            if not (0 <= b < e <= len(rec.tokens)):
                raise _err(ErrorCode.InvalidArgument, "bad forward range")
            self._advance_committed(rec)
            if rec.committed_hint < b:
                raise _err(ErrorCode.MissingKV, f"position {rec.committed_hint} is empty before "
                                                f"prefill begin {b}")
            if rec.alloc_len < e:
                raise _err(ErrorCode.Internal, "forward range not allocated")
            if rec.fold_frontier > b or rec.digest_len > b:
                raise _err(ErrorCode.Internal, "fold/digest beyond range")
            fold_from = rec.fold_frontier
            slots = [self._resolve(rec, pos) for pos in range(fold_from, e)]
            digests = []
            while rec.digest_len < e:
                rec.prefix_digest = hm.extend_prefix_digest(rec.prefix_digest,
                                                            rec.tokens[rec.digest_len])
                rec.digest_len += 1
                if rec.digest_len > b:
                    digests.append(rec.prefix_digest)
            plan.entries.append({"seq": ent.seq, "range": (b, e), "fold_from": fold_from,
                                 "slots": slots, "digests": digests})
            plan.total_outputs += e - b
        keep = []
        for (seq, rng, dest, addr, tag) in self.pending:
            if seq not in seen:
                keep.append((seq, rng, dest, addr, tag))
                continue
            rec = self._get(seq)
            plan.sends.append({"seq": seq, "range": rng, "dest": dest, "dest_addr": addr,
                               "user_tag": tag,
                               "slots": [self._resolve(rec, p) for p in range(*rng)]})
        self.pending = keep
        return plan

    # -- computation stage --------------------------------------------------------------
    def Attention(self, layer, plan, hidden_in, sink=None):  # kv_cache.cc:308-371
        if not (layer == plan.next_layer and layer < self.layers):
            raise _err(ErrorCode.LayerOrderViolation,
                       f"expected layer {plan.next_layer}, got {layer}")
        hidden_in = [int(x) for x in hidden_in]
        if len(hidden_in) != plan.total_outputs:
            raise _err(ErrorCode.Internal, "hidden input size mismatch")
        out = [0] * plan.total_outputs
        idx = 0
        for ent in plan.entries:
            rec = self._get(ent["seq"])
            s = rec.fold_sums[layer]
            b, e = ent["range"]
            for pos in range(ent["fold_from"], e):
                pg, sl = ent["slots"][pos - ent["fold_from"]]
                if pos >= b:
                    if self.fill[pg, sl, layer] == 0:
                        self.values[pg, sl, layer] = hm.kv_entry_words(
                            ent["digests"][pos - b], layer, self.dim)
                        self.fill[pg, sl, layer] = 1
                    s = (s + hm.entry_digest(self.values[pg, sl, layer])) & M64
                    x = hidden_in[idx]
                    out[idx] = hm.next_hidden(x, hm.attention_out(x, pos + 1, s))
                    idx += 1
                else:
                    if self.fill[pg, sl, layer] == 0:
                        raise _err(ErrorCode.MissingKV, "fold over empty slot")
                    s = (s + hm.entry_digest(self.values[pg, sl, layer])) & M64
            rec.fold_sums[layer] = s
            if layer == self.layers - 1:
                rec.fold_frontier = e
                self._advance_committed(rec)
        for snd in plan.sends:
            rows = []
            for (pg, sl) in snd["slots"]:
                if self.fill[pg, sl, layer] == 0:
                    raise _err(ErrorCode.MissingKV, "sending empty slot")
                rows.append(self.values[pg, sl, layer])
            payload = np.concatenate(rows) if rows else np.zeros(0, np.uint64)
            if sink is not None:
                sink(layer, {k: snd[k] for k in ("seq", "range", "dest", "dest_addr", "user_tag")},
                     payload)
        plan.next_layer += 1
        return np.asarray(out, dtype=np.uint64)

    def GatherRange(self, seq, token_range, layer):  # kv_cache.cc:373-387
        rec = self._get(seq)
        rows = []
        for pos in range(*token_range):
            pg, sl = self._resolve(rec, pos)
            if self.fill[pg, sl, layer] == 0:
                raise _err(ErrorCode.MissingKV, "gather over empty slot")
            rows.append(self.values[pg, sl, layer])
        return np.concatenate(rows) if rows else np.zeros(0, np.uint64)

    def BuildAddr(self, seq, token_range):  # kv_cache.cc:389-407
        rec = self._get(seq)
        b, e = token_range
        if b < rec.fork_len:
            raise _err(ErrorCode.InvalidArgument, "address must cover own slots only")
        ranges = []
        for pos in range(b, e):
            pg, sl = self._resolve(rec, pos)
            if ranges and ranges[-1][0] == pg and ranges[-1][1] + ranges[-1][2] == sl:
                ranges[-1] = (pg, ranges[-1][1], ranges[-1][2] + 1)
            else:
                ranges.append((pg, sl, 1))
        a = KVAddrInfo(ranges, b, e - b)
        addr_validate(a)
        return a

    # -- transfer agent -----------------------------------------------------------------
    def ApplyRemoteWrite(self, addr, layer, payload, tag):  # kv_cache.cc:409-463
        payload = np.asarray(payload, dtype=np.uint64)
        if len(payload) != addr.token_count * self.dim:
            raise _err(ErrorCode.InvalidArgument, "payload size mismatch")
        owner = -1
        for (p, b, c) in addr.ranges:
            if p < 0 or p >= self.num_pages or self.owner[p] < 0:
                return ApplyStatus.UnknownAddress
            if owner == -1:
                owner = self.owner[p]
            if self.owner[p] != owner:
                return ApplyStatus.UnknownAddress
            for s in range(b, b + c):
                if s < 0 or s >= self.page_size or not self.expecting[p, s]:
                    return ApplyStatus.UnknownAddress
        rec = self.records.get(owner)
        if rec is None or rec.window is None:
            return ApplyStatus.UnknownAddress
        w = rec.window
        key = (tag, layer, addr.token_begin)
        if key in w.applied:
            return ApplyStatus.Duplicate
        w.applied.add(key)
        word = 0
        for (p, b, c) in addr.ranges:
            for s in range(b, b + c):
                if self.fill[p, s, layer] == 0:
                    self.values[p, s, layer] = payload[word:word + self.dim]
                    self.fill[p, s, layer] = 2
                word += self.dim
                w.received += 1
        if not w.complete and w.received >= w.expected:
            w.complete = True
            self.completed.append(owner)
        return ApplyStatus.Ok

    def DrainReceiveCompletions(self):  # kv_cache.cc:465-480
        done, self.completed = self.completed, []
        for seq in done:
            rec = self.records.get(seq)
            if rec is None:
                continue
            self._advance_committed(rec)
            rec.finished = True
            self.CommitToTree(seq)
        return done

    # -- lifecycle ---------------------------------------------------------------------------
    def SetFinished(self, seq, finished):
        self._get(seq).finished = bool(finished)

    def CommitToTree(self, seq):  # kv_cache.cc:484-490
        rec = self._get(seq)
        self._advance_committed(rec)
        n = min(rec.committed_hint, len(rec.tokens))
        if n > 0:
            self.tree.Insert(rec.tokens[:n], seq)

    def FreeSequence(self, seq):  # kv_cache.cc:492-518
        rec = self._get(seq)
        if rec.refcount != 0:
            raise _err(ErrorCode.Internal, "freeing a sequence with live children")
        rec.window = None
        for pg in rec.own_pages:
            self.owner[pg] = -1
            self.expecting[pg] = 0
            self.fill[pg] = 0
            self.free_pages.append(pg)
        if rec.parent >= 0 and rec.parent in self.records:
            self.records[rec.parent].refcount -= 1
        self.pending = [p for p in self.pending if p[0] != seq]
        self.tree.Remove(seq)
        del self.records[seq]

    def BytesPerPage(self):
        return self.page_size * self.layers * self.dim * 8

    def Evict(self, bytes_needed):  # kv_cache.cc:520-546
        if bytes_needed <= 0:
            return 0
        freed = 0
        while len(self.free_pages) * self.BytesPerPage() < bytes_needed:
            victim = -1
            for seq in self.tree.SequencesByLru():
                rec = self.records.get(seq)
                if rec is None or not rec.finished or rec.refcount != 0 or not rec.own_pages:
                    continue
                if self.tree.HasPinnedNode(seq):
                    continue
                victim = seq
                break
            if victim < 0:
                raise _err(ErrorCode.CannotEvict, "all remaining sequences are pinned or live")
            rec = self.records[victim]
            freed += max(0, min(len(rec.tokens), rec.alloc_len) - rec.fork_len)
            self.FreeSequence(victim)
        return freed

    def Pin(self, prefix, flag):
        self.tree.Pin(prefix, flag)

    # -- queries ------------------------------------------------------------------------------
    def HasSequence(self, seq):
        return seq in self.records

    def GetRecord(self, seq) -> SequenceRecordInfo:
        r = self._get(seq)
        win = None
        if r.window is not None:
            win = {"range": r.window.range, "expected_writes": r.window.expected,
                   "received_writes": r.window.received, "complete": r.window.complete}
        return SequenceRecordInfo(r.id, r.parent, r.fork_len, r.refcount, r.finished,
                                  r.alloc_len, r.committed_hint, len(r.tokens),
                                  list(r.own_pages), r.fold_frontier, r.digest_len,
                                  r.prefix_digest, win)

    def Committed(self, seq):
        rec = self._get(seq)
        self._advance_committed(rec)
        return rec.committed_hint

    def ReadEntryWords(self, seq, pos, layer):
        pg, sl = self._resolve(self._get(seq), pos)
        return self.values[pg, sl, layer].copy()

    def FillOf(self, seq, pos, layer):
        pg, sl = self._resolve(self._get(seq), pos)
        return FillState(int(self.fill[pg, sl, layer]))

    def FreePages(self):
        return len(self.free_pages)

    def TotalPages(self):
        return self.num_pages

    def SequenceCount(self):
        return len(self.records)

    def SequenceIds(self):
        return sorted(self.records)

    def PendingSendCount(self):
        return len(self.pending)

    def TreeNodeCount(self):
        return self.tree.NodeCount()

    def TreeContains(self, seq):
        return self.tree.Contains(seq)

    def TreeLastTouch(self, seq):
        return self.tree.LastTouch(seq)

    def TreeSequencesByLru(self):
        return self.tree.SequencesByLru()
