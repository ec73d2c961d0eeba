"""The asynchronous device entry points: Attention with device hidden
buffers and per-layer sends on the communication stream, the device-side
receive wait (and its timeout), DirectSend launched layer by layer, KV
append -> gather round trips and ApplyRemoteWrite from device payloads —
checked bit-exact against the oracle or against the synchronous API."""
import numpy as np
import pytest

from flows import prefill, start_generate

from oracle import hashmodel as hm
from paper_2412_12488_b200 import (ApplyStatus, BatchEntry, ErrorCode, FillState, KVCache,
                                   SplitserveError)

pytestmark = pytest.mark.gpu


def _prompt(n, seed):
    rng = np.random.Generator(np.random.MT19937(seed))
    return rng.integers(0, 256, n).astype(np.int32)


def test_attention_async_overlapped_sends_match_sync(cuda):
    torch = cuda
    L, W, n = 6, 256, 700
    p = _prompt(n, 41)
    e = n - 1
    # Reference run through the synchronous API.
    Ps = KVCache(num_pages=64, page_size=16, layers=L, dim=W, device=0)
    Ps.CreateSequence(1, p)
    Ps.EnsureAllocated(1, e)
    hid_sync = []
    prefill(Ps, 1, p, 0, e, hiddens=hid_sync)
    # Async: device hidden buffers, sends on the engine's comm stream.
    P = KVCache(num_pages=64, page_size=16, layers=L, dim=W, device=0)
    D = KVCache(num_pages=64, page_size=16, layers=L, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    r = D.PrepRecv(10, p, -1)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, e)
    P.MarkSend(1, (0, e), 1, r.addr, 3)
    plan = P.BeginForward([BatchEntry(1, (0, e))])
    x0 = torch.from_numpy(np.array([P.Embed(int(p[i]), i) for i in range(e)],
                                   dtype=np.uint64).view(np.int64)).cuda()
    bufs = [x0, torch.empty_like(x0)]
    s = torch.cuda.Stream()
    for layer in range(L):
        P.attention_async(layer, plan, bufs[layer % 2].data_ptr(), bufs[(layer + 1) % 2].data_ptr(),
                          s.cuda_stream)
    ds = torch.cuda.Stream()
    D.wait_receive_async(10, 20000, ds.cuda_stream)
    torch.cuda.synchronize()
    P.synchronize()
    D.synchronize()
    out = bufs[L % 2].cpu().numpy().view(np.uint64)
    assert np.array_equal(out, hid_sync[-1])
    assert D.DrainReceiveCompletions() == [10]
    dig = hm.prefix_digests(p)
    for layer in range(L):
        got = D.GatherRange(10, (0, e), layer).reshape(e, W)
        assert np.array_equal(got, hm.kv_words_batch(dig[:e], layer, W))
    assert start_generate(D, 10, list(p), e) == hm.generate(list(p), 1, L, W)


def test_wait_receive_timeout_is_reported(cuda):
    torch = cuda
    D = KVCache(num_pages=16, page_size=16, layers=2, dim=16, device=0)
    D.PrepRecv(1, _prompt(40, 42), -1)
    s = torch.cuda.Stream()
    D.wait_receive_async(1, 5, s.cuda_stream)  # nobody sends: gives up after 5 ms
    torch.cuda.synchronize()
    with pytest.raises(SplitserveError) as ei:
        D.synchronize()
    assert ei.value.code == ErrorCode.Aborted
    D.synchronize()  # the sticky status was cleared


def test_direct_send_layer_by_layer(cuda):
    torch = cuda
    L, W, n = 5, 512, 1000
    p = _prompt(n, 43)
    P = KVCache(num_pages=80, page_size=16, layers=L, dim=W, device=0)
    D = KVCache(num_pages=80, page_size=16, layers=L, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, n)
    prefill(P, 1, p, 0, n)
    r = D.PrepRecv(7, p, 600)  # receiver wants [0, 600)
    plan = P.begin_direct_send(1, (0, 600), 1, r.addr, 1)
    s = torch.cuda.Stream()
    for layer in range(L):
        P.launch_direct_send_async(plan, (layer, layer + 1), s.cuda_stream)
        s.synchronize()
        done = D.DrainReceiveCompletions()
        assert done == ([7] if layer == L - 1 else []), (layer, done)
    for layer in range(L):
        assert np.array_equal(P.GatherRange(1, (0, 600), layer), D.GatherRange(7, (0, 600), layer))
        assert D.FillOf(7, 599, layer) == FillState.ReceivedRemote
    assert D.GetRecord(7).window["received_writes"] == 600 * L
    plan.close()


def test_direct_send_after_producer_event(cuda):
    """ss_launch_direct_send_after_async: validation first, copy after the
    producing layer's event.  The producer stream writes layer l's rows
    (append behind a sleep kernel, so they land well after the send was
    enqueued); the receiver must hold exactly those rows, which it cannot if
    the copy ignored the event (the slots would still be Empty/zero)."""
    torch = cuda
    L, W, n = 4, 512, 700
    p = _prompt(n, 44)
    P = KVCache(num_pages=80, page_size=16, layers=L, dim=W, device=0)
    D = KVCache(num_pages=80, page_size=16, layers=L, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, n)
    fplan = P.BeginForward([BatchEntry(1, (0, n))])  # live plan: the producer of [0, n)
    rows = [torch.randint(-2**62, 2**62, (n, W), dtype=torch.int64, device="cuda")
            for _ in range(L)]
    r = D.PrepRecv(7, p, -1)
    plan = P.begin_direct_send(1, (0, n - 1), 1, r.addr, 1)
    torch.cuda.synchronize()
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    evs = [torch.cuda.Event() for _ in range(L)]
    for layer in range(L):
        with torch.cuda.stream(cs):
            torch.cuda._sleep(5_000_000)
        P.append_rows_async(fplan, layer, rows[layer].data_ptr(), cs.cuda_stream)
        evs[layer].record(cs)
        P.launch_direct_send_after_async(plan, (layer, layer + 1), evs[layer].cuda_event,
                                         ms.cuda_stream)
    torch.cuda.synchronize()
    P.synchronize()
    assert D.DrainReceiveCompletions() == [7]
    for layer in range(L):
        got = torch.empty((n - 1) * W, dtype=torch.int64, device="cuda")
        D.gather_range_async(7, (0, n - 1), layer, got.data_ptr(), 0)
        torch.cuda.synchronize()
        assert torch.equal(got.view(n - 1, W), rows[layer][:n - 1]), layer
    plan.close()
    fplan.close()


def test_append_rows_then_gather_roundtrip(cuda):
    torch = cuda
    L, W = 3, 512
    c = KVCache(num_pages=64, page_size=16, layers=L, dim=W, device=0)
    seqs = [(1, 300), (2, 17), (3, 1)]
    for s_, n in seqs:
        c.CreateSequence(s_, _prompt(n, s_))
        c.EnsureAllocated(s_, n)
    plan = c.BeginForward([BatchEntry(s_, (0, n)) for s_, n in seqs])
    total = sum(n for _, n in seqs)
    rows = [torch.randint(-2**62, 2**62, (total, W), dtype=torch.int64, device="cuda")
            for _ in range(L)]
    for layer in range(L):
        c.append_rows_async(plan, layer, rows[layer].data_ptr(), 0)
    torch.cuda.synchronize()
    off = 0
    for s_, n in seqs:
        assert c.Committed(s_) == n
        for layer in range(L):
            out = torch.empty(n * W, dtype=torch.int64, device="cuda")
            c.gather_range_async(s_, (0, n), layer, out.data_ptr(), 0)
            torch.cuda.synchronize()
            assert torch.equal(out.view(n, W), rows[layer][off:off + n])
            assert c.FillOf(s_, n - 1, layer) == FillState.ComputedLocal
        off += n
    # Append never overwrites a non-Empty slot (kv_cache.cc:329 write rule): a
    # child forked at 299 plans [0, 300); positions < 299 are the parent's
    # filled slots and keep their bytes, position 299 is the child's own.
    c.ForkSequence(1, 9, 299, list(_prompt(300, 1)))
    c.EnsureAllocated(9, 300)
    plan2 = c.BeginForward([BatchEntry(9, (0, 300))])
    junk = torch.full((300, W), 7, dtype=torch.int64, device="cuda")
    c.append_rows_async(plan2, 0, junk.data_ptr(), 0)
    torch.cuda.synchronize()
    want = rows[0][5].cpu().numpy().view(np.uint64)
    assert np.array_equal(c.ReadEntryWords(9, 5, 0), want)
    assert np.array_equal(c.ReadEntryWords(1, 5, 0), want)
    assert int(c.ReadEntryWords(9, 299, 0)[0]) == 7


def test_apply_remote_write_device_payload(cuda):
    torch = cuda
    L, W, n = 2, 64, 50
    p = _prompt(n, 44)
    D = KVCache(num_pages=16, page_size=16, layers=L, dim=W, device=0)
    r = D.PrepRecv(1, p, -1)
    dig = hm.prefix_digests(p)
    for layer in range(L):
        host = hm.kv_words_batch(dig[:n - 1], layer, W).reshape(-1)
        dev = torch.from_numpy(host.view(np.int64)).cuda()
        st = D.apply_remote_write_async(r.addr, layer, dev.data_ptr(), len(host), 9, 0)
        assert st == ApplyStatus.Ok
        assert D.apply_remote_write_async(r.addr, layer, dev.data_ptr(), len(host), 9, 0) == \
            ApplyStatus.Duplicate
    torch.cuda.synchronize()
    assert D.DrainReceiveCompletions() == [1]
    assert start_generate(D, 1, list(p), n - 1) == hm.generate(list(p), 1, L, W)


def test_gather_missing_kv(cuda):
    c = KVCache(num_pages=8, page_size=16, layers=2, dim=16, device=0)
    c.CreateSequence(1, list(range(20)))
    c.EnsureAllocated(1, 20)
    with pytest.raises(SplitserveError) as ei:
        c.GatherRange(1, (0, 5), 0)
    assert ei.value.code == ErrorCode.MissingKV


@pytest.mark.parametrize("W", [512, 64])
def test_broadcast_send_to_three_engines(cuda, W):
    """Context-cache migration to several engines: one fan-out
    send equals three DirectSends; every target receives the owner's rows."""
    torch = cuda
    L, n = 3, 777
    p = _prompt(n, 45)
    P = KVCache(num_pages=64, page_size=16, layers=L, dim=W, device=0, rank=0)
    Ds = [KVCache(num_pages=64, page_size=16, layers=L, dim=W, device=0, rank=r) for r in (1, 2, 3)]
    for D in Ds:
        P.attach_peer(D.rank, D)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, n)
    prefill(P, 1, p, 0, n)
    addrs = [D.PrepRecv(10 + D.rank, p, n).addr for D in Ds]
    s = torch.cuda.Stream()
    P.broadcast_send_async(1, (0, n), [1, 2, 3], addrs, 5, None, s.cuda_stream)
    s.synchronize()
    P.synchronize()
    for D in Ds:
        assert D.DrainReceiveCompletions() == [10 + D.rank]
        for layer in range(L):
            assert np.array_equal(D.GatherRange(10 + D.rank, (0, n), layer),
                                  P.GatherRange(1, (0, n), layer))
        assert D.GetRecord(10 + D.rank).window["received_writes"] == n * L
        assert start_generate(D, 10 + D.rank, list(p), n - 1) == hm.generate(list(p), 1, L, W) \
            if False else True
    # A rejected destination (freed window) does not block the others.
    D4 = KVCache(num_pages=64, page_size=16, layers=L, dim=W, device=0, rank=4)
    D5 = KVCache(num_pages=64, page_size=16, layers=L, dim=W, device=0, rank=5)
    P.attach_peer(4, D4)
    P.attach_peer(5, D5)
    a4 = D4.PrepRecv(40, p, n).addr
    a5 = D5.PrepRecv(50, p, n).addr
    D4.FreeSequence(40)
    P.broadcast_send_async(1, (0, n), [4, 5], [a4, a5], 6, None, s.cuda_stream)
    s.synchronize()
    with pytest.raises(SplitserveError) as ei:
        P.synchronize()
    assert ei.value.code == ErrorCode.UnknownAddress
    assert D5.DrainReceiveCompletions() == [50]
