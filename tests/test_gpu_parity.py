"""GPU parity: the B200 library against the CPU oracle (restatement, pinned
to the reference) and, where its .so travelled, the compiled reference —
bit-exact KV page contents, fill states, page tables, addresses, match
lengths, hidden outputs and tokens."""
import json
from pathlib import Path

import numpy as np
import pytest

from flows import one_p_one_d, prefill, start_generate
from scenarios import make_script, run_script

from oracle import hashmodel as hm
from oracle.kvcache_oracle import KVCache as OracleCache
from paper_2412_12488_b200 import (ApplyStatus, BatchEntry, ErrorCode, FillState, KVAddrInfo,
                                   KVCache, SplitserveError)

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def _j(log):
    return json.loads(json.dumps(log, default=lambda o: list(o) if isinstance(o, tuple) else str(o)))


def _prompt(n, seed=1, vocab=256):
    rng = np.random.Generator(np.random.MT19937(seed))
    return [int(x) for x in rng.integers(0, vocab, n)]


def _gpu(**k):
    k.setdefault("device", 0)
    return KVCache(**k)


def _check_all_kv(E, seq, prompt, n, layers, dim):
    """Every (position, layer) entry of seq equals the oracle's KvEntryWords."""
    dig = hm.prefix_digests(prompt[:n])
    for layer in range(layers):
        got = E.GatherRange(seq, (0, n), layer).reshape(n, dim)
        want = hm.kv_words_batch(dig, layer, dim)
        bad = np.nonzero((got != want).any(axis=1))[0]
        assert bad.size == 0, f"layer {layer}: {bad.size} rows differ, first at {bad[:5]}"


# ---------------------------------------------------------------------------
# Golden fixtures and op scripts
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("via", ["sink", "peer"])
def test_tiny_1p1d_matches_golden(cuda, via):
    g = json.loads((GOLD / "tiny_1p1d.json").read_text())
    c = g["config"]
    P = _gpu(num_pages=c["num_pages"], page_size=c["page_size"], layers=c["layers"], dim=c["dim"])
    D = _gpu(num_pages=c["num_pages"], page_size=c["page_size"], layers=c["layers"], dim=c["dim"],
             rank=1)
    if via == "peer":
        P.attach_peer(1, D)
    hid = []
    r = one_p_one_d(P, D, g["prompt"], c["end"], via=via, hiddens=hid, max_tokens=3)
    assert r["done"] == g["completions"]
    assert r["match_len"] == g["match_len"]
    assert [list(x) for x in r["addr"].ranges] == g["addr"]["ranges"]
    assert r["tokens"] == g["tokens"]
    assert [str(int(x)) for x in hid[-1]] == g["p_hidden_last_layer"]
    assert [str(int(x)) for x in hid[0][:8]] == g["p_hidden_layer0_first8"]
    assert D.GetRecord(10).own_pages == g["d_own_pages"]
    assert D.Committed(10) == g["d_committed"]
    assert [int(D.FillOf(10, 0, l)) for l in range(c["layers"])] == g["d_fill_pos0"]
    assert [int(D.FillOf(10, 511, l)) for l in range(c["layers"])] == g["d_fill_pos511"]
    assert [str(int(x)) for x in D.ReadEntryWords(10, 0, 0)] == g["d_entry_pos0_layer0"]
    import hashlib

    h = hashlib.sha256()
    for pos in range(c["prompt_len"]):
        for layer in range(c["layers"]):
            h.update(D.ReadEntryWords(10, pos, layer).astype("<u8").tobytes())
    assert h.hexdigest() == g["d_entries_sha256"]
    assert P.FreePages() == g["p_free_pages"] and D.FreePages() == g["d_free_pages"]


@pytest.mark.parametrize("seed", range(4))
def test_scripts_match_golden(cuda, seed):
    g = json.loads((GOLD / "scripts.json").read_text())[str(seed)]
    c = _gpu(num_pages=24, page_size=4, layers=2, dim=8)
    assert _j(run_script(c, make_script(seed, n_ops=80, data=True))) == g


@pytest.mark.parametrize("seed", range(10, 16))
def test_scripts_match_restatement(cuda, seed):
    ops = make_script(seed, n_ops=120, data=True)
    a = run_script(_gpu(num_pages=24, page_size=4, layers=2, dim=8), ops)
    b = run_script(OracleCache(num_pages=24, page_size=4, layers=2, dim=8), ops)
    assert _j(a) == _j(b)


@pytest.mark.parametrize("seed", range(20, 23))
def test_scripts_match_reference(cuda, ref_lib, seed):
    ops = make_script(seed, n_ops=120, data=True)
    a = run_script(_gpu(num_pages=24, page_size=4, layers=2, dim=8), ops)
    b = run_script(KVCache(num_pages=24, page_size=4, layers=2, dim=8, lib=ref_lib), ops)
    assert _j(a) == _j(b)


# ---------------------------------------------------------------------------
# Known answers (SPEC.md examples) on the device path
# ---------------------------------------------------------------------------
def _commit_prefix(E, seq, tokens):
    E.CreateSequence(seq, tokens)
    E.EnsureAllocated(seq, len(tokens))
    prefill(E, seq, tokens, 0, len(tokens))
    E.SetFinished(seq, True)
    E.CommitToTree(seq)


def test_prep_recv_after_cached_prefix(cuda):
    # cache holds tokens[:16] of a 64-token prompt -> m=16, 48 slots, 3 fresh pages.
    p = _prompt(64, 3)
    D = _gpu(num_pages=32, page_size=16, layers=2, dim=16)
    _commit_prefix(D, 1, p[:16])
    r = D.PrepRecv(2, p, 64)
    assert r.match_len == 16 and r.addr.token_count == 48
    assert r.addr.ranges == [(1, 0, 16), (2, 0, 16), (3, 0, 16)]
    assert D.GetRecord(2).parent == 1 and D.GetRecord(1).refcount == 1


def test_fork_relative_paging(cuda):
    # a child forked at m=5 starts at slot 0 of a fresh page.
    p = _prompt(23, 4)
    D = _gpu(num_pages=32, page_size=16, layers=2, dim=16)
    _commit_prefix(D, 1, p[:5])
    r = D.PrepRecv(2, p, 23)
    assert r.match_len == 5
    assert r.addr.ToJson() == '{"ranges":[[1,0,16],[2,0,2]],"token_begin":5,"token_count":18}'


def test_partial_edge_match_and_remove_quirk(cuda):
    # SURVEY.md A.3 + A.4.
    D = _gpu(num_pages=32, page_size=4, layers=1, dim=8)
    _commit_prefix(D, 10, [5, 6, 7, 8])
    assert D.MatchPrefix([5, 6, 9]) == 2
    E = _gpu(num_pages=32, page_size=4, layers=1, dim=8)
    _commit_prefix(E, 10, [1, 2, 3])
    _commit_prefix(E, 11, [1, 2, 3])
    E.FreeSequence(11)
    assert E.MatchPrefix([1, 2, 3]) == 0 and E.TreeNodeCount() == 0 and E.TreeContains(10)


def test_fully_matched_prep_recv_forks_without_window(cuda):
    # SURVEY.md A.5.
    p = _prompt(40, 5)
    D = _gpu(num_pages=32, page_size=16, layers=2, dim=16)
    _commit_prefix(D, 1, p)
    r = D.PrepRecv(2, p, 40)
    assert r.match_len == 40 and r.addr.token_count == 0 and r.addr.ranges == []
    rec = D.GetRecord(2)
    assert rec.window is None and rec.parent == 1 and D.GetRecord(1).refcount == 1


# ---------------------------------------------------------------------------
# Microserving flows against the oracle
# ---------------------------------------------------------------------------
def test_8b_shape_1p1d_peer_bit_exact(cuda):
    """configs[1]: Llama-3.1-8B KV shape (L=32, W=512 = 4 KiB/token/layer),
    4K prompt, prep_recv end=-1, device-direct remote_send."""
    L, W, n = 32, 512, 4096
    p = _prompt(n, 11)
    P = _gpu(num_pages=n // 16 + 8, page_size=16, layers=L, dim=W)
    D = _gpu(num_pages=n // 16 + 8, page_size=16, layers=L, dim=W, rank=1)
    P.attach_peer(1, D)
    r = one_p_one_d(P, D, p, -1, via="peer", max_tokens=2)
    assert r["done"] == [10] and r["addr"].token_count == n - 1
    _check_all_kv(D, 10, p, n, L, W)
    for pos in (0, n - 2):
        assert D.FillOf(10, pos, 0) == FillState.ReceivedRemote
    assert D.FillOf(10, n - 1, L - 1) == FillState.ComputedLocal
    assert r["tokens"] == hm.generate(p, 2, L, W)


@pytest.mark.parametrize("ratio", [0.1, 0.2, 0.3])
def test_balanced_pd(cuda, ratio):
    """D prefills the tail prompt[s:]; P sends [0, s)."""
    L, W, n = 4, 128, 700
    p = _prompt(n, 12)
    s = int((1 - ratio) * n)
    P = _gpu(num_pages=64, page_size=16, layers=L, dim=W)
    D = _gpu(num_pages=64, page_size=16, layers=L, dim=W, rank=1)
    P.attach_peer(1, D)
    r = one_p_one_d(P, D, p, s, via="peer", max_tokens=2)
    assert r["end"] == s
    assert r["tokens"] == hm.generate(p, 2, L, W)
    _check_all_kv(D, 10, p, n, L, W)


def test_context_cache_forked_prefix(cuda):
    """PAPER.md Fig 4: D holds a 60-token context; prep_recv matches it, P
    sends only the rest, D's fork reuses the prefix pages."""
    L, W = 3, 64
    p = _prompt(200, 13)
    P = _gpu(num_pages=64, page_size=16, layers=L, dim=W)
    D = _gpu(num_pages=64, page_size=16, layers=L, dim=W, rank=1)
    P.attach_peer(1, D)
    _commit_prefix(D, 1, p[:60])
    r = one_p_one_d(P, D, p, -1, via="peer")
    assert r["match_len"] == 60
    assert r["tokens"] == hm.generate(p, 1, L, W)
    _check_all_kv(D, 10, p, 200, L, W)


def test_case1_directsend_plus_prefill_then_send(cuda):
    """SPEC.md:271 Case 1: sender matched 600, receiver asks [200, 999):
    DirectSend [200, 600) + PrefillThenSend [600, 999)."""
    L, W, n = 3, 64, 1000
    p = _prompt(n, 14)
    P = _gpu(num_pages=160, page_size=16, layers=L, dim=W)
    D = _gpu(num_pages=160, page_size=16, layers=L, dim=W, rank=1)
    P.attach_peer(1, D)
    _commit_prefix(P, 1, p[:600])
    _commit_prefix(D, 2, p[:200])
    r = D.PrepRecv(10, p, 999)
    assert r.match_len == 200 and r.addr.token_count == 799
    P.ForkSequence(1, 20, 600, p)
    P.EnsureAllocated(20, 999)
    P.direct_send_async(20, (200, 600), 1, r.addr.Slice(200, 600), 9)
    P.MarkSend(20, (600, 999), 1, r.addr.Slice(600, 999), 9)
    prefill(P, 20, p, 600, 999)
    P.synchronize()
    assert D.DrainReceiveCompletions() == [10]
    assert start_generate(D, 10, p, 999) == hm.generate(p, 1, L, W)
    _check_all_kv(D, 10, p, n, L, W)


def test_case2_prefill_only_gap(cuda):
    """SPEC.md:272 Case 2: sender matched 200, receiver asks [600, 999):
    PrefillOnly [200, 600) + PrefillThenSend [600, 999)."""
    L, W, n = 3, 64, 1000
    p = _prompt(n, 15)
    P = _gpu(num_pages=160, page_size=16, layers=L, dim=W)
    D = _gpu(num_pages=160, page_size=16, layers=L, dim=W, rank=1)
    P.attach_peer(1, D)
    _commit_prefix(P, 1, p[:200])
    _commit_prefix(D, 2, p[:600])
    r = D.PrepRecv(10, p, 999)
    assert r.match_len == 600
    P.ForkSequence(1, 20, 200, p)
    P.EnsureAllocated(20, 999)
    P.MarkSend(20, (600, 999), 1, r.addr, 3)
    prefill(P, 20, p, 200, 999)
    P.synchronize()
    assert D.DrainReceiveCompletions() == [10]
    assert start_generate(D, 10, p, 999, 3) == hm.generate(p, 3, L, W)


def test_multi_frame_chunked_apply_and_dedupe(cuda):
    """kv_cache.cc:438-457: frames dedupe by (tag, layer, token_begin) and may
    arrive in arbitrary chunks; completion counts every addressed slot."""
    L, W, n = 2, 32, 100
    p = _prompt(n, 16)
    D = _gpu(num_pages=16, page_size=16, layers=L, dim=W)
    Ref = OracleCache(num_pages=16, page_size=16, layers=L, dim=W)
    outs = []
    for E in (D, Ref):
        r = E.PrepRecv(1, p, -1)
        dig = hm.prefix_digests(p)
        log = []
        for layer in range(L):
            for (b, e) in ((0, 30), (30, 31), (31, 99)):
                sub = r.addr.Slice(b, e)
                pl = hm.kv_words_batch(dig[b:e], layer, W).reshape(-1)
                log.append(int(E.ApplyRemoteWrite(sub, layer, pl, 5)))
            log.append(int(E.ApplyRemoteWrite(r.addr.Slice(0, 30), layer,
                                               np.zeros(30 * W, np.uint64), 5)))
        bad = KVAddrInfo([(15, 0, 1)], 0, 1)
        log.append(int(E.ApplyRemoteWrite(bad, 0, np.zeros(W, np.uint64), 5)))
        with pytest.raises(SplitserveError) as ei:
            E.ApplyRemoteWrite(r.addr, 0, np.zeros(3, np.uint64), 5)
        assert ei.value.code == ErrorCode.InvalidArgument
        log.append(tuple(E.DrainReceiveCompletions()))
        log.append(E.GetRecord(1).window)
        outs.append(log)
    assert outs[0] == outs[1]
    assert outs[0][3] == int(ApplyStatus.Duplicate)
    _check_all_kv(D, 1, p, n - 1, L, W)


def test_missing_kv_before_transfer_completes(cuda):
    """SPEC.md:280 protocol-order safety: start_generate before the transfer
    completes is MissingKV, never wrong tokens."""
    p = _prompt(50, 17)
    D = _gpu(num_pages=16, page_size=16, layers=2, dim=16)
    D.PrepRecv(1, p, -1)
    D.EnsureAllocated(1, 50)
    with pytest.raises(SplitserveError) as ei:
        D.BeginForward([BatchEntry(1, (49, 50))])
    assert ei.value.code == ErrorCode.MissingKV


def test_layer_order_violation(cuda):
    p = _prompt(10, 18)
    E = _gpu(num_pages=8, page_size=16, layers=3, dim=16)
    E.CreateSequence(1, p)
    E.EnsureAllocated(1, 10)
    plan = E.BeginForward([BatchEntry(1, (0, 10))])
    x = np.zeros(10, np.uint64)
    with pytest.raises(SplitserveError) as ei:
        E.Attention(1, plan, x)
    assert ei.value.code == ErrorCode.LayerOrderViolation


def test_corrupted_transfer_diverges(cuda):
    """SPEC.md:304 no-recompute: a corrupted transferred entry changes the
    generated tokens (the receiver really reads what arrived)."""
    L, W, n = 2, 16, 64
    p = _prompt(n, 19)
    diverged = 0
    for trial in range(8):
        P = _gpu(num_pages=16, page_size=16, layers=L, dim=W)
        D = _gpu(num_pages=16, page_size=16, layers=L, dim=W, rank=1)

        def corrupt(layer, send, payload, trial=trial):
            if layer == trial % L:
                payload[(trial * 37) % len(payload)] ^= np.uint64(1 << (trial % 64))
            return payload

        r = one_p_one_d(P, D, p, -1, via="sink", corrupt=corrupt, max_tokens=3)
        diverged += r["tokens"] != hm.generate(p, 3, L, W)
    assert diverged >= 7


def test_directsend_to_freed_window_is_rejected(cuda):
    L, W, n = 2, 64, 80
    p = _prompt(n, 20)
    P = _gpu(num_pages=16, page_size=16, layers=L, dim=W)
    D = _gpu(num_pages=16, page_size=16, layers=L, dim=W, rank=1)
    P.attach_peer(1, D)
    _commit_prefix(P, 1, p)
    r = D.PrepRecv(5, p, -1)
    D.FreeSequence(5)
    P.direct_send_async(1, (0, n - 1), 1, r.addr, 1)
    with pytest.raises(SplitserveError) as ei:
        P.synchronize()
    assert ei.value.code == ErrorCode.UnknownAddress
    D.PrepRecv(6, p, -1)
    assert D.GetRecord(6).window["received_writes"] == 0


def test_70b_shape_directsend_bit_exact(cuda):
    """The bench's migration at the 70B KV shape (W=512, 8K tokens), reduced
    to 8 layers: D's received rows equal P's, window accounting completes."""
    L, W, n = 8, 512, 8192
    p = _prompt(n, 21)
    P = _gpu(num_pages=n // 16 + 8, page_size=16, layers=L, dim=W)
    D = _gpu(num_pages=n // 16 + 8, page_size=16, layers=L, dim=W, rank=1)
    P.attach_peer(1, D)
    _commit_prefix(P, 1, p)
    for rep in range(2):
        r = D.PrepRecv(100 + rep, p, -1)
        P.direct_send_async(1, (0, n - 1), 1, r.addr, rep)
        P.synchronize()
        assert D.DrainReceiveCompletions() == [100 + rep]
        for layer in range(L):
            assert np.array_equal(P.GatherRange(1, (0, n - 1), layer),
                                  D.GatherRange(100 + rep, (0, n - 1), layer))
        assert D.Committed(100 + rep) == n - 1
        assert start_generate(D, 100 + rep, p, n - 1) == hm.generate(p, 1, L, W)
        D.FreeSequence(100 + rep)
