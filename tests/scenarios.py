"""Deterministic op scripts over the KVCache interface, with an observable log.

The same script is applied to the product library, the compiled reference
(oracle/_ref) and the Python restatement; parity = identical logs.  Ops
cover the reference's declaration/lifecycle surface (kv_cache.h:136-235):
PrepRecv (with prefix matches -> forks), CreateSequence, ForkSequence,
EnsureAllocated, receive of a whole window through ApplyRemoteWrite with
the oracle's KV words, DrainReceiveCompletions, a forward pass
(BeginForward + Attention), CommitToTree, SetFinished, FreeSequence, Evict,
Pin, MatchPrefix.  Errors are logged by ErrorCode name, so error paths are
compared too.
"""
from __future__ import annotations

import random

import numpy as np

from paper_2412_12488_b200 import BatchEntry, SplitserveError

from oracle import hashmodel as hm


def make_script(seed: int, n_ops: int = 120, data: bool = True, vocab: int = 8):
    """Random but reproducible op list.  Prompts come from a few families
    sharing prefixes so the radix tree sees matches, partial edges and splits."""
    rnd = random.Random(seed)
    fams = [[rnd.randrange(vocab) for _ in range(60)] for _ in range(3)]

    def prompt():
        f = rnd.choice(fams)
        k = rnd.randrange(1, 60)
        tail = [rnd.randrange(vocab) for _ in range(rnd.randrange(0, 20))]
        return f[:k] + tail

    ops, next_id = [], 1
    for _ in range(n_ops):
        kinds = ["prep", "create", "fork", "ensure", "free", "match", "pin", "evict", "finish",
                 "commit", "append"]
        if data:
            kinds += ["recv", "recv", "forward", "forward"]
        k = rnd.choice(kinds)
        sid = rnd.randrange(1, max(2, next_id))
        if k == "prep":
            p = prompt()
            ops.append(("prep", next_id, p, rnd.choice([-1, len(p), max(1, len(p) // 2)])))
            next_id += 1
        elif k == "create":
            ops.append(("create", next_id, prompt()))
            next_id += 1
        elif k == "fork":
            ops.append(("fork", sid, next_id, rnd.randrange(0, 30)))
            next_id += 1
        elif k == "ensure":
            ops.append(("ensure", sid, rnd.randrange(0, 80)))
        elif k == "free":
            ops.append(("free", sid))
        elif k == "match":
            ops.append(("match", prompt()))
        elif k == "pin":
            ops.append(("pin", prompt()[: rnd.randrange(1, 30)], rnd.random() < 0.7))
        elif k == "evict":
            ops.append(("evict", rnd.choice([0, 1, 4096, 40000, 200000])))
        elif k == "finish":
            ops.append(("finish", sid, rnd.random() < 0.8))
        elif k == "commit":
            ops.append(("commit", sid))
        elif k == "append":
            ops.append(("append", sid, rnd.randrange(vocab)))
        elif k == "recv":
            ops.append(("recv", sid, rnd.randrange(1 << 30)))
        elif k == "forward":
            ops.append(("forward", sid, rnd.randrange(0, 40), rnd.randrange(1, 30)))
    return ops


def _snapshot(c, ids):
    out = {"free": c.FreePages(), "nseq": c.SequenceCount(), "nodes": c.TreeNodeCount()}
    recs = {}
    for s in ids:
        if c.HasSequence(s):
            r = c.GetRecord(s)
            recs[s] = (r.parent, r.fork_len, r.refcount, r.finished, r.alloc_len,
                       r.committed_hint, r.num_tokens, tuple(r.own_pages), r.fold_frontier,
                       r.digest_len, None if r.window is None else
                       (tuple(r.window["range"]), r.window["expected_writes"],
                        r.window["received_writes"], r.window["complete"]))
    out["recs"] = recs
    out["lru"] = c.TreeSequencesByLru()
    return out


def _err(e: SplitserveError):
    return ("ERR", e.name)


def run_script(c, ops, seed=0):
    """Applies ops to cache `c`; returns the observable log."""
    log, tokens_of = [], {}
    for op in ops:
        kind = op[0]
        try:
            if kind == "prep":
                _, s, p, end = op
                r = c.PrepRecv(s, p, end)
                tokens_of[s] = list(p)
                res = ("ok", r.match_len, r.addr.token_begin, r.addr.token_count,
                       tuple(map(tuple, r.addr.ranges)))
            elif kind == "create":
                _, s, p = op
                c.CreateSequence(s, p)
                tokens_of[s] = list(p)
                res = ("ok",)
            elif kind == "fork":
                _, parent, child, fl = op
                c.ForkSequence(parent, child, fl)
                if parent in tokens_of:
                    tokens_of[child] = tokens_of[parent][:fl]
                res = ("ok",)
            elif kind == "ensure":
                _, s, upto = op
                c.EnsureAllocated(s, upto)
                res = ("ok",)
            elif kind == "free":
                c.FreeSequence(op[1])
                res = ("ok",)
            elif kind == "match":
                res = ("ok",) + tuple(c.MatchPrefixSeq(op[1]))
            elif kind == "pin":
                c.Pin(op[1], op[2])
                res = ("ok",)
            elif kind == "evict":
                res = ("ok", c.Evict(op[1]))
            elif kind == "finish":
                c.SetFinished(op[1], op[2])
                res = ("ok",)
            elif kind == "commit":
                c.CommitToTree(op[1])
                res = ("ok",)
            elif kind == "append":
                c.AppendToken(op[1], op[2])
                if op[1] in tokens_of:
                    tokens_of[op[1]].append(op[2])
                res = ("ok",)
            elif kind == "recv":
                res = _recv_window(c, op[1], op[2], tokens_of)
            elif kind == "forward":
                res = _forward(c, op[1], op[2], op[3], tokens_of)
            else:
                raise AssertionError(kind)
        except SplitserveError as e:
            res = _err(e)
        ids = sorted(set(x for o in ops for x in o[1:3] if isinstance(x, int)))
        log.append((op[0], res, _snapshot(c, [i for i in ids if i < 10_000])))
    return log


def _recv_window(c, s, tag, tokens_of):
    """Receive the sequence's open window (all layers) with the oracle's KV words."""
    r = c.GetRecord(s)
    if r.window is None or r.window["complete"]:
        return ("skip",)
    b, e = r.window["range"]
    addr = c.BuildAddr(s, (b, e))
    dig = hm.prefix_digests(tokens_of[s][:e], c.hash_seed)[b:e]
    sts = []
    for layer in range(c.layers):
        payload = hm.kv_words_batch(dig, layer, c.dim).reshape(-1)
        sts.append(int(c.ApplyRemoteWrite(addr, layer, payload, tag)))
    dup = int(c.ApplyRemoteWrite(addr, 0, hm.kv_words_batch(dig, 0, c.dim).reshape(-1), tag))
    done = c.DrainReceiveCompletions()
    return ("ok", tuple(sts), dup, tuple(done))


def _forward(c, s, begin_hint, count, tokens_of):
    """A forward pass over [b, b+count) clipped to the sequence: EnsureAllocated,
    BeginForward, Attention for every layer; logs the last hidden word."""
    if not c.HasSequence(s):
        c.GetRecord(s)  # raises UnknownSequence like the reference would
    r = c.GetRecord(s)
    n = r.num_tokens
    b = min(max(r.fold_frontier, r.committed_hint, 0), n)
    e = min(n, b + count)
    if e <= b:
        return ("skip",)
    c.EnsureAllocated(s, e)
    plan = c.BeginForward([BatchEntry(s, (b, e))])
    toks = tokens_of.get(s)
    x = np.array([c.Embed(toks[i] if toks else 0, i) for i in range(b, e)], dtype=np.uint64)
    for layer in range(c.layers):
        x = c.Attention(layer, plan, x)
    if hasattr(plan, "close"):
        plan.close()
    return ("ok", b, e, int(x[-1]))
