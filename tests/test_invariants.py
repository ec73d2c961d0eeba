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
  committed = f, and its first f positions resolve to the parent's slots
  (host-only scripts reach f = 0 only; test_gpu_parity forks past it);
* window accounting: an open receive window over [m, e) expects (e - m) * L
  writes, and its address round-trips through the JSON and binary codecs.
"""
import pytest

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


@pytest.mark.parametrize("seed", range(6))
def test_invariants_hold_after_every_op(seed):
    L, P = 2, 4
    c = KVCache(num_pages=24, page_size=P, layers=L, dim=8, device=-1)
    tokens_of = {}
    checked = {"match": 0, "fork": 0, "window": 0}
    for op in make_script(300 + seed, n_ops=200, data=False):
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
                    span = (0, fl)
                    assert c.BuildAddr(parent, span).slots(P) == c.BuildAddr(child, span).slots(P)
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
        except SplitserveError:
            pass  # error paths are compared with the reference in test_host_bookkeeping
        for s in list(tokens_of):
            if not c.HasSequence(s):
                tokens_of.pop(s)
        _check_pages(c)
    # (Forks past position 0 need committed KV, i.e. a data path: host-only
    # scripts exercise them at fork_len 0; test_gpu_parity covers the rest.)
    assert checked["match"] > 0 and checked["window"] > 0, checked
