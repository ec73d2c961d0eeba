"""SPEC.md's invariants ("prefix soundness vs brute-force LCP,
page accounting, fork transparency, address round-trip") checked after every
op of the random scripts of tests/scenarios.py, on the product library's
host side (host-only cache, CPU):

* page accounting: free pages + every sequence's own pages == total pages,
  and no page is owned twice;
* prefix soundness: a MatchPrefixSeq(q) of length m names a sequence whose
  first m tokens are q[:m], and m never exceeds the longest common prefix of
  q with any live sequence's tokens (brute force);
* fork transparency: a child forked at f has parent, fork_len = f and
  committed = f, and its first f positions read the parent's stored words
  (host-only scripts reach f = 0 only; a directed device test forks past it);
* window accounting: an open receive window over [m, e) expects (e - m) * L
  writes, and its address round-trips through the JSON and binary codecs.
"""
import pytest

import scenarios
from scenarios import make_script

from paper_2412_12488_b200 import KVAddrInfo, KVCache, SplitserveError


def _lcp(a, b):
    n = 0
    for x, y in zip(a, b):
        if x != y:
            break
        n += 1
    return n


def _check_pages(c):
    owned = []
    for s in c.SequenceIds():
        owned += c.GetRecord(s).own_pages
    assert len(owned) == len(set(owned)), "a page owned twice"
    assert c.FreePages() + len(owned) == c.TotalPages()


def _run(c, ops, L, P):
    tokens_of = {}
    checked = {"match": 0, "fork": 0, "fork_past0": 0, "window": 0}
    for op in ops:
        kind = op[0]
        try:
            if kind == "prep":
                _, s, p, end = op
                r = c.PrepRecv(s, p, end)
                tokens_of[s] = list(p)
                rec = c.GetRecord(s)
                if r.addr.token_count > 0 and rec.window is not None:
                    b, e = rec.window["range"]
                    assert (b, e) == (r.match_len, r.match_len + r.addr.token_count)
                    assert rec.window["expected_writes"] == (e - b) * L
                    assert KVAddrInfo.FromJson(r.addr.ToJson()) == r.addr
                    assert KVAddrInfo.DecodeFrom(r.addr.EncodeTo())[0] == r.addr
                    checked["window"] += 1
            elif kind == "create":
                c.CreateSequence(op[1], op[2])
                tokens_of[op[1]] = list(op[2])
            elif kind == "fork":
                _, parent, child, fl = op
                c.ForkSequence(parent, child, fl)
                if parent in tokens_of:
                    tokens_of[child] = tokens_of[parent][:fl]
                rec = c.GetRecord(child)
                if fl > 0:
                    assert rec.parent == parent and rec.fork_len == fl
                else:  # a fork at 0 shares nothing: the reference links no parent
                    assert rec.fork_len == 0 and rec.parent in (-1, parent)
                assert c.Committed(child) == fl
                if fl > 0:
                    checked["fork_past0"] += 1
                checked["fork"] += 1
            elif kind == "ensure":
                c.EnsureAllocated(op[1], op[2])
            elif kind == "free":
                c.FreeSequence(op[1])
                tokens_of.pop(op[1], None)
            elif kind == "match":
                q = list(op[1])
                m, ref = c.MatchPrefixSeq(q)
                live = [t for s, t in tokens_of.items() if c.HasSequence(s)]
                assert m <= max([_lcp(q, t) for t in live], default=0)
                if m > 0 and ref in tokens_of:
                    assert tokens_of[ref][:m] == q[:m]
                checked["match"] += 1
            elif kind == "pin":
                c.Pin(op[1], op[2])
            elif kind == "evict":
                c.Evict(op[1])
            elif kind == "finish":
                c.SetFinished(op[1], op[2])
            elif kind == "commit":
                c.CommitToTree(op[1])
            elif kind == "append":
                c.AppendToken(op[1], op[2])
                if op[1] in tokens_of:
                    tokens_of[op[1]].append(op[2])
            elif kind == "recv":
                scenarios._recv_window(c, op[1], op[2], tokens_of)
            elif kind == "forward":
                scenarios._forward(c, op[1], op[2], op[3], tokens_of)
        except SplitserveError:
            pass  # error paths are compared with the reference in test_host_bookkeeping
        for s in list(tokens_of):
            if not c.HasSequence(s):
                tokens_of.pop(s)
        _check_pages(c)
    return checked


@pytest.mark.parametrize("seed", range(6))
def test_invariants_hold_after_every_op(seed):
    L, P = 2, 4
    c = KVCache(num_pages=24, page_size=P, layers=L, dim=8, device=-1)
    checked = _run(c, make_script(300 + seed, n_ops=200, data=False), L, P)
    # (Forks past position 0 need committed KV, i.e. a data path: host-only
    # scripts reach them at fork_len 0; the device variant below goes past.)
    assert checked["match"] > 0 and checked["window"] > 0, checked


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4))
def test_invariants_with_device_data(cuda, seed):
    """The same checks on a device cache with the data path (receives
    through ApplyRemoteWrite, forward passes): sequences commit KV, so
    forks past position 0 and cached-prefix PrepRecvs occur."""
    L, P = 2, 4
    c = KVCache(num_pages=32, page_size=P, layers=L, dim=8, device=0)
    checked = _run(c, make_script(400 + seed, n_ops=200, data=True), L, P)
    assert checked["match"] > 0 and checked["window"] > 0, checked


@pytest.mark.gpu
def test_fork_transparency_past_zero(cuda):
    """Forks of a sequence with committed KV at page-aligned and unaligned
    lengths: the child's record, committed frontier, slots and stored words
    for [0, f) are the parent's (the random scripts rarely commit before a
    fork)."""
    import numpy as np

    from paper_2412_12488_b200 import BatchEntry

    L, P = 2, 4
    c = KVCache(num_pages=64, page_size=P, layers=L, dim=8, device=0)
    toks = [(7 * i + 3) % 13 for i in range(39)]
    c.CreateSequence(1, toks)
    c.EnsureAllocated(1, len(toks))
    plan = c.BeginForward([BatchEntry(1, (0, len(toks)))])
    x = np.array([c.Embed(t, i) for i, t in enumerate(toks)], dtype=np.uint64)
    for layer in range(L):
        x = c.Attention(layer, plan, x)
    plan.close()
    c.synchronize()
    assert c.Committed(1) == len(toks)
    for fl in (1, 4, 5, 16, 38, 39):  # unaligned and page-aligned (P = 4)
        child = 100 + fl
        c.ForkSequence(1, child, fl)
        rec = c.GetRecord(child)
        assert rec.parent == 1 and rec.fork_len == fl and c.Committed(child) == fl
        # (BuildAddr covers a sequence's own slots only, as in the reference:
        # the shared part is compared through the stored words.)
        for pos in {0, fl // 2, fl - 1}:
            for layer in range(L):
                assert np.array_equal(c.ReadEntryWords(1, pos, layer),
                                      c.ReadEntryWords(child, pos, layer))
        _check_pages(c)
