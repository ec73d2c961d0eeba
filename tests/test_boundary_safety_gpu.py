"""Safety of the device-direct boundary (round-2 advisor findings):

* a destination address that does not give one slot per sent row is
  rejected (DirectSend / BroadcastSend raise like the reference's frame
  decode, kv_addr.cc:16-30; a MarkSend'ed one is rejected by the receiver's
  validation) and no receiver slot is written;
* the MissingKV scan of a gather keeps the sticky asynchronous error bits
  (a rejected async send is still reported by Synchronize);
* Synchronize / internal work are ordered after EVERY caller stream used;
* device receive windows are recycled once drained (a long-running decode
  engine keeps finished sequences cached), exhaustion is a retryable
  OutOfPages raised before any state change, and a stale sender into a
  drained window is rejected instead of counting into the row's next
  window.
"""
import numpy as np
import pytest

from flows import prefill

from paper_2412_12488_b200 import BatchEntry, ErrorCode, KVAddrInfo, KVCache, SplitserveError

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["inline", "grid"])
def validation(request, monkeypatch):
    """Both validation paths of a device-direct send: inside the copy grid
    (small addresses, the default) and a separate validation grid."""
    monkeypatch.setenv("MICROKV_INLINE_VALIDATE_SLOTS", "2048" if request.param == "inline" else "0")
    return request.param


def _prompt(n, seed):
    return np.random.Generator(np.random.MT19937(seed)).integers(0, 256, n).astype(np.int32)


def _pair(L=2, W=128, pages=64):
    P = KVCache(num_pages=pages, page_size=16, layers=L, dim=W, device=0)
    D = KVCache(num_pages=pages, page_size=16, layers=L, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    return P, D


def test_direct_send_rejects_short_address(cuda, validation):
    P, D = _pair()
    p = _prompt(100, 1)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, 100)
    prefill(P, 1, p, 0, 100)
    r = D.PrepRecv(7, p, 40)  # 40 slots
    # Claims 40 tokens but its ranges cover 16: the copy would read
    # destination slots past the list.
    short = KVAddrInfo([(r.addr.ranges[0][0], 0, 16)], 0, 40)
    with pytest.raises(SplitserveError) as ei:
        P.begin_direct_send(1, (0, 40), 1, short, 1)
    assert ei.value.code == ErrorCode.AddrMismatch
    overlap = KVAddrInfo([(r.addr.ranges[0][0], 0, 16), (r.addr.ranges[0][0], 8, 16),
                          (r.addr.ranges[1][0], 0, 8)], 0, 40)
    with pytest.raises(SplitserveError) as ei:
        P.begin_direct_send(1, (0, 40), 1, overlap, 1)
    assert ei.value.code == ErrorCode.InvalidArgument
    with pytest.raises(SplitserveError) as ei:
        P.broadcast_send_async(1, (0, 40), [1], [short], 1, None, 0)
    assert ei.value.code == ErrorCode.AddrMismatch
    # Nothing landed; the window still opens normally with a valid address.
    assert D.FillOf(7, 0, 0) == 0
    P.direct_send_async(1, (0, 40), 1, r.addr, 1, (0, 2), 0)
    P.synchronize()
    assert D.DrainReceiveCompletions() == [7]


def test_marked_send_with_malformed_address_is_rejected_by_receiver(cuda, validation):
    """MarkSend keeps the reference's checks only; the plan's send of a
    malformed address is rejected by the receiver-side validation (sticky
    UnknownAddress at Synchronize) and writes nothing."""
    P, D = _pair()
    p = _prompt(64, 2)
    r_other = D.PrepRecv(5, _prompt(48, 3), -1)  # another sequence's window on D
    r = D.PrepRecv(7, p, 40)
    bad = KVAddrInfo([(r.addr.ranges[0][0], 0, 16)], 0, 40)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, 64)
    P.MarkSend(1, (0, 40), 1, bad, 3)
    plan = P.BeginForward([BatchEntry(1, (0, 64))])
    h = np.array([P.Embed(int(p[i]), i) for i in range(64)], dtype=np.uint64)
    for layer in range(2):
        h = P.Attention(layer, plan, h)
    with pytest.raises(SplitserveError) as ei:
        P.synchronize()
    assert ei.value.code == ErrorCode.UnknownAddress
    assert D.DrainReceiveCompletions() == []
    for seq, n in ((7, 40), (5, r_other.addr.token_count)):
        for layer in range(2):
            assert D.FillOf(seq, 0, layer) == 0 and D.FillOf(seq, n - 1, layer) == 0
    plan.close()


def test_missing_kv_scan_keeps_sticky_async_error(cuda, validation):
    torch = cuda
    P, D = _pair()
    p = _prompt(64, 4)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, 64)
    prefill(P, 1, p, 0, 64)
    r = D.PrepRecv(7, p, 32)
    plan = P.begin_direct_send(1, (0, 32), 1, r.addr, 1)
    D.FreeSequence(7)  # the window is gone: the async send will be rejected
    P.launch_direct_send_async(plan, (0, 2), 0)
    torch.cuda.synchronize()
    # A gather whose fill must be proven on the device (a sequence with
    # uncommitted positions) runs the MissingKV scan on P ...
    P.CreateSequence(2, p)
    P.EnsureAllocated(2, 64)
    out = torch.empty(16 * 128, dtype=torch.int64, device="cuda")
    with pytest.raises(SplitserveError) as ei:
        P.gather_range_async(2, (0, 16), 0, out.data_ptr(), 0)
    assert ei.value.code == ErrorCode.MissingKV
    # ... and the earlier rejection is still reported.
    with pytest.raises(SplitserveError) as ei:
        P.synchronize()
    assert ei.value.code == ErrorCode.UnknownAddress
    plan.close()


def test_synchronize_waits_for_every_caller_stream(cuda):
    torch = cuda
    L, W, n = 2, 512, 256
    c = KVCache(num_pages=32, page_size=16, layers=L, dim=W, device=0)
    c.CreateSequence(1, _prompt(n, 5))
    c.EnsureAllocated(1, n)
    plan = c.BeginForward([BatchEntry(1, (0, n))])
    rows = torch.randint(-2**62, 2**62, (n * W,), dtype=torch.int64, device="cuda")
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(a):
        torch.cuda._sleep(200_000_000)  # ~0.1 s
    c.append_rows_async(plan, 0, rows.data_ptr(), a.cuda_stream)
    done_a = torch.cuda.Event()
    done_a.record(a)
    c.append_rows_async(plan, 1, rows.data_ptr(), b.cuda_stream)  # stream B used last
    c.synchronize()
    assert done_a.query(), "Synchronize returned before stream A's queued append"
    # Internal work (the plan free) is ordered after both streams as well.
    plan.close()
    assert c.Committed(1) == n


def test_window_rows_recycled_after_drain(cuda):
    """More receives than device window rows, each finished sequence kept
    cached (never freed): works because drained windows give their row back."""
    P, D = _pair(L=1, W=128, pages=4200)
    p = _prompt(3, 6)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, 3)
    prefill(P, 1, p, 0, 3)
    for i in range(4100):
        toks = np.array([i // 256, i % 256, 0], np.int32)  # no prompt fully cached
        r = D.PrepRecv(10 + i, toks, -1)
        assert r.match_len < 2
        P.direct_send_async(1, (r.match_len, 2), 1, r.addr, i, (0, 1), 0)
        P.synchronize()
        assert D.DrainReceiveCompletions() == [10 + i]
    assert D.SequenceCount() == 4100


def test_window_exhaustion_is_retryable_and_atomic(cuda):
    D = KVCache(num_pages=4200, page_size=16, layers=1, dim=128, device=0)
    for i in range(4096):
        D.PrepRecv(10 + i, np.array([i % 256, i // 256, 1], np.int32), -1)
    free = D.FreePages()
    with pytest.raises(SplitserveError) as ei:
        D.PrepRecv(99999, np.array([7, 7, 7], np.int32), -1)
    assert ei.value.code == ErrorCode.OutOfPages and ei.value.retryable
    assert D.FreePages() == free and not D.HasSequence(99999)
    D.FreeSequence(10)
    D.PrepRecv(99999, np.array([7, 7, 7], np.int32), -1)


def test_stale_sender_into_drained_window_is_rejected(cuda, validation):
    P, D = _pair()
    p = _prompt(64, 7)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, 64)
    prefill(P, 1, p, 0, 64)
    r = D.PrepRecv(7, p, 32)
    plan = P.begin_direct_send(1, (0, 32), 1, r.addr, 1)
    P.launch_direct_send_async(plan, (0, 2), 0)
    P.synchronize()
    assert D.DrainReceiveCompletions() == [7]
    # The window's row goes to the next receive; a stale re-send of the old
    # address must not count into it.
    r2 = D.PrepRecv(8, _prompt(40, 8), -1)
    P.launch_direct_send_async(plan, (0, 2), 0)
    with pytest.raises(SplitserveError) as ei:
        P.synchronize()
    assert ei.value.code == ErrorCode.UnknownAddress
    assert D.DrainReceiveCompletions() == []
    assert D.GetRecord(8).window["received_writes"] == 0
    # The receiver's own data is untouched and seq 7 stays complete.
    assert np.array_equal(P.GatherRange(1, (0, 32), 1), D.GatherRange(7, (0, 32), 1))
    plan.close()
    del r2


def test_stale_plan_after_window_reopen_is_rejected(cuda):
    """Later launches of a plan skip the validation grid and check the
    receiver window's open-generation: after the receiver frees the sequence
    and re-opens a window — the same window id over the same pages, LIFO —
    the plan's next layer is rejected and writes nothing."""
    P, D = _pair(L=4)
    p = _prompt(64, 9)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, 64)
    prefill(P, 1, p, 0, 64)
    r = D.PrepRecv(7, p, 48)
    plan = P.begin_direct_send(1, (0, 48), 1, r.addr, 1)
    P.launch_direct_send_async(plan, (0, 1), 0)   # validates the address
    P.launch_direct_send_async(plan, (1, 2), 0)   # generation check, same window: lands
    P.synchronize()
    assert all(int(D.FillOf(7, pos, l)) == 2 for pos in (0, 47) for l in (0, 1))  # ReceivedRemote
    D.FreeSequence(7)
    r2 = D.PrepRecv(8, p, 48)                     # the same pages (LIFO order) and window row
    assert sorted(x[0] for x in r2.addr.ranges) == sorted(x[0] for x in r.addr.ranges)
    P.launch_direct_send_async(plan, (2, 3), 0)   # stale: the window was re-opened
    with pytest.raises(SplitserveError) as ei:
        P.synchronize()
    assert ei.value.code == ErrorCode.UnknownAddress
    assert all(int(D.FillOf(8, pos, l)) == 0 for pos in range(48) for l in range(4))
    plan.close()
