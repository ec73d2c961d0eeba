"""ss_append_rows_send_async: the KV append fused with remote_send.  One
launch per layer must leave exactly the state of the unfused pair
(append_rows_async, then a DirectSend of the layer: kv_cache.cc:328-367) —
the sender's pages and fill states, the receiver's pages, fill states and
per-layer window counters — bit-exact, including ranges inside a batched
plan, rows whose local slot was already written (sent from the page, not
from the dense buffer), a receiver that already holds some slots, the
toy-model rows of the oracle, and a rejected address."""
import numpy as np
import pytest

from oracle import hashmodel as hm
from paper_2412_12488_b200 import BatchEntry, ErrorCode, FillState, KVCache, SplitserveError

pytestmark = pytest.mark.gpu


def _prompt(n, seed):
    rng = np.random.Generator(np.random.MT19937(seed))
    return rng.integers(0, 256, n).astype(np.int32)


def _pair(L, W, pages=96):
    P = KVCache(num_pages=pages, page_size=16, layers=L, dim=W, device=0)
    D = KVCache(num_pages=pages, page_size=16, layers=L, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    return P, D


def _layer_rows(torch, seq_cache, seq, rng_range, layer, W):
    b, e = rng_range
    out = torch.empty((e - b) * W, dtype=torch.int64, device="cuda")
    seq_cache.gather_range_async(seq, (b, e), layer, out.data_ptr(), 0)
    torch.cuda.synchronize()
    return out.view(e - b, W)


@pytest.mark.parametrize("W", [512, 128])
def test_fused_equals_append_then_send(cuda, W):
    torch = cuda
    L, n = 4, 1000
    p = _prompt(n, 61)
    rows = torch.randint(-2**62, 2**62, (L, n, W), dtype=torch.int64, device="cuda")
    results = []
    for fused in (False, True):
        P, D = _pair(L, W)
        P.CreateSequence(1, p)
        P.EnsureAllocated(1, n)
        fplan = P.BeginForward([BatchEntry(1, (0, n))])
        r = D.PrepRecv(7, p, -1)
        splan = P.begin_direct_send(1, (0, n - 1), 1, r.addr, 3)
        s = torch.cuda.Stream()
        for layer in range(L):
            if fused:
                P.append_rows_send_async(fplan, splan, (layer, layer + 1), rows[layer].data_ptr(),
                                         s.cuda_stream)
            else:
                P.append_rows_async(fplan, layer, rows[layer].data_ptr(), s.cuda_stream)
                P.launch_direct_send_async(splan, (layer, layer + 1), s.cuda_stream)
        s.synchronize()
        P.synchronize()
        assert D.DrainReceiveCompletions() == [7]
        st = {"P": [_layer_rows(torch, P, 1, (0, n), l, W).cpu() for l in range(L)],
              "D": [_layer_rows(torch, D, 7, (0, n - 1), l, W).cpu() for l in range(L)],
              "Pfill": [P.FillOf(1, pos, l) for l in range(L) for pos in (0, 517, n - 1)],
              "Dfill": [D.FillOf(7, pos, l) for l in range(L) for pos in (0, 517, n - 2)],
              "win": D.GetRecord(7).window["received_writes"]}
        results.append(st)
        fplan.close()
        splan.close()
    a, b = results
    for l in range(L):
        assert torch.equal(a["P"][l], b["P"][l])
        assert torch.equal(a["D"][l], b["D"][l])
        assert torch.equal(b["D"][l], rows[l, :n - 1].cpu())
    assert a["Pfill"] == b["Pfill"] and set(b["Pfill"]) == {FillState.ComputedLocal}
    assert a["Dfill"] == b["Dfill"] and set(b["Dfill"]) == {FillState.ReceivedRemote}
    assert a["win"] == b["win"] == (n - 1) * L


def test_fused_range_inside_batched_plan_and_layer_ready_flags(cuda):
    """The send covers the tail of the second entry of a two-sequence plan;
    the receiver's per-layer wait releases layer by layer."""
    torch = cuda
    L, W = 3, 512
    pa, pb = _prompt(300, 62), _prompt(800, 63)
    P, D = _pair(L, W)
    P.CreateSequence(1, pa)
    P.EnsureAllocated(1, 300)
    P.CreateSequence(2, pb)
    P.EnsureAllocated(2, 800)
    fplan = P.BeginForward([BatchEntry(1, (0, 300)), BatchEntry(2, (0, 800))])
    total = 1100
    rows = torch.randint(-2**62, 2**62, (L, total, W), dtype=torch.int64, device="cuda")
    # The receiver already holds [0, 256) of pb (a cached prefix): it asks for [256, 799).
    D.CreateSequence(5, pb[:256])
    D.EnsureAllocated(5, 256)
    fp5 = D.BeginForward([BatchEntry(5, (0, 256))])
    seed_rows = torch.randint(-2**62, 2**62, (L, 256, W), dtype=torch.int64, device="cuda")
    for l in range(L):
        D.append_rows_async(fp5, l, seed_rows[l].data_ptr(), 0)
    torch.cuda.synchronize()
    fp5.close()
    D.SetFinished(5, True)
    D.CommitToTree(5)
    r = D.PrepRecv(9, pb, -1)
    m = r.match_len
    assert m == 256
    splan = P.begin_direct_send(2, (m, 799), 1, r.addr, 4)
    s, ws = torch.cuda.Stream(), torch.cuda.Stream()
    for layer in range(L):
        P.append_rows_send_async(fplan, splan, (layer, layer + 1), rows[layer].data_ptr(),
                                 s.cuda_stream)
        D.wait_receive_layer_async(9, layer, 20000, ws.cuda_stream)
    torch.cuda.synchronize()
    P.synchronize()
    D.synchronize()
    assert D.DrainReceiveCompletions() == [9]
    for layer in range(L):
        got = _layer_rows(torch, D, 9, (m, 799), layer, W)
        assert torch.equal(got, rows[layer, 300 + m:300 + 799])
        got_p = _layer_rows(torch, P, 1, (0, 300), layer, W)
        assert torch.equal(got_p, rows[layer, :300])
    fplan.close()
    splan.close()


def test_fused_sends_existing_local_rows_from_the_page(cuda):
    """Positions whose local slot already holds KV — here [0, 200) received
    from a third engine before P prefills [0, n) — keep their contents
    (Empty-only write rule) and the receiver gets those contents, as the
    reference's send reads the pool after the write (kv_cache.cc:328-367)."""
    torch = cuda
    L, W, n = 2, 512, 400
    p = _prompt(n, 64)
    P, D = _pair(L, W)
    E = KVCache(num_pages=96, page_size=16, layers=L, dim=W, device=0, rank=2)
    E.attach_peer(0, P)
    first = torch.randint(-2**62, 2**62, (L, 200, W), dtype=torch.int64, device="cuda")
    E.CreateSequence(1, p)
    E.EnsureAllocated(1, 200)
    fe = E.BeginForward([BatchEntry(1, (0, 200))])
    for l in range(L):
        E.append_rows_async(fe, l, first[l].data_ptr(), 0)
    rp = P.PrepRecv(1, p, 200)
    E.direct_send_async(1, (0, 200), 0, rp.addr, 1, (0, L), 0)
    torch.cuda.synchronize()
    E.synchronize()
    fe.close()
    assert P.DrainReceiveCompletions() == [1]
    P.EnsureAllocated(1, n)
    second = torch.randint(-2**62, 2**62, (L, n, W), dtype=torch.int64, device="cuda")
    f2 = P.BeginForward([BatchEntry(1, (0, n))])
    r = D.PrepRecv(3, p, -1)
    splan = P.begin_direct_send(1, (0, n - 1), 1, r.addr, 5)
    for l in range(L):
        P.append_rows_send_async(f2, splan, (l, l + 1), second[l].data_ptr(), 0)
    torch.cuda.synchronize()
    P.synchronize()
    assert D.DrainReceiveCompletions() == [3]
    for l in range(L):
        want = torch.cat([first[l], second[l, 200:n - 1]])
        assert torch.equal(_layer_rows(torch, D, 3, (0, n - 1), l, W), want)
        assert torch.equal(_layer_rows(torch, P, 1, (0, n - 1), l, W), want)
        assert P.FillOf(1, 10, l) == FillState.ReceivedRemote
        assert P.FillOf(1, 300, l) == FillState.ComputedLocal
    f2.close()
    splan.close()


def test_fused_all_layers_one_launch_toy_rows_match_oracle(cuda):
    """Oracle rows (KvEntryWords of the prompt's prefix digests) appended and
    sent for every layer in one launch: the receiver's pages equal the
    oracle's words bit for bit."""
    torch = cuda
    L, W, n = 4, 128, 513
    p = _prompt(n, 65)
    P, D = _pair(L, W)
    e = n - 1
    dig = hm.prefix_digests(list(p))
    rows = np.stack([hm.kv_words_batch(dig[:e], l, W).reshape(e, W) for l in range(L)])
    rows_t = torch.from_numpy(rows.view(np.int64)).cuda()
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, e)
    fplan = P.BeginForward([BatchEntry(1, (0, e))])
    r = D.PrepRecv(4, p, -1)
    splan = P.begin_direct_send(1, (0, e), 1, r.addr, 6)
    P.append_rows_send_async(fplan, splan, (0, L), rows_t.data_ptr(), 0)
    torch.cuda.synchronize()
    P.synchronize()
    assert D.DrainReceiveCompletions() == [4]
    for l in range(L):
        assert np.array_equal(D.GatherRange(4, (0, e), l).reshape(e, W), rows[l])
        for pos in (0, 255, e - 1):
            assert np.array_equal(D.ReadEntryWords(4, pos, l), hm.kv_entry_words(int(dig[pos]), l, W))
    fplan.close()
    splan.close()


def test_fused_rejected_address_writes_nothing_remote(cuda):
    """The receiver's window is freed before the launch: validation rejects
    the address, nothing lands remote, the local append still happens and
    ss_synchronize reports UnknownAddress."""
    torch = cuda
    L, W, n = 2, 512, 300
    p = _prompt(n, 66)
    P, D = _pair(L, W)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, n)
    fplan = P.BeginForward([BatchEntry(1, (0, n))])
    r = D.PrepRecv(2, p, -1)
    splan = P.begin_direct_send(1, (0, n - 1), 1, r.addr, 7)
    D.FreeSequence(2)
    rows = torch.randint(-2**62, 2**62, (L, n, W), dtype=torch.int64, device="cuda")
    P.append_rows_send_async(fplan, splan, (0, L), rows.data_ptr(), 0)
    torch.cuda.synchronize()
    with pytest.raises(SplitserveError) as ei:
        P.synchronize()
    assert ei.value.code == ErrorCode.UnknownAddress
    for l in range(L):
        assert torch.equal(_layer_rows(torch, P, 1, (0, n), l, W), rows[l])
    assert D.DrainReceiveCompletions() == []
    fplan.close()
    splan.close()


def test_fused_send_range_outside_the_plan_is_rejected(cuda):
    L, W, n = 2, 512, 300
    p = _prompt(n, 67)
    P, D = _pair(L, W)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, n)
    fplan = P.BeginForward([BatchEntry(1, (0, 200))])  # outputs [0, 200) only
    r = D.PrepRecv(2, p, -1)
    splan = P.begin_direct_send(1, (0, n - 1), 1, r.addr, 7)
    with pytest.raises(SplitserveError) as ei:
        P.append_rows_send_async(fplan, splan, (0, 1), 0, 0)
    assert ei.value.code == ErrorCode.InvalidArgument
    fplan.close()
    splan.close()
