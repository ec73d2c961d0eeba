"""DirectSend row movers (ss_set_send_mode): the copy kernel on an SM budget
(grid capped at a few CTAs, as a send overlapping the next prefill layer
runs) and the copy-engine mover (batched 3-D copies + a fill/counter
kernel).  Both must leave the receiver bit-identical to the oracle's
KvEntryWords, including when the sender's and the receiver's page
boundaries do not line up (the receiver forked a cached prefix at a
position that is not a page multiple), and both reject a bad address."""
import numpy as np
import pytest

from flows import prefill, start_generate

from oracle import hashmodel as hm
from paper_2412_12488_b200 import ErrorCode, KVCache, SplitserveError

pytestmark = pytest.mark.gpu

L, W, PAGE = 32, 512, 16  # Llama-3.1-8B KV shape


def _prompt(n, seed):
    return np.random.Generator(np.random.MT19937(seed)).integers(0, 256, n).astype(np.int32)


def _engines(n):
    P = KVCache(num_pages=n // PAGE + 8, page_size=PAGE, layers=L, dim=W, device=0, rank=0)
    D = KVCache(num_pages=2 * (n // PAGE) + 16, page_size=PAGE, layers=L, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    return P, D


def _check(torch, D, seq, p, lo, hi):
    dig = hm.prefix_digests(p)
    out = torch.empty((hi - lo) * W, dtype=torch.int64, device="cuda")
    for layer in range(L):
        D.gather_range_async(seq, (lo, hi), layer, out.data_ptr(), 0)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint64).reshape(hi - lo, W)
        assert np.array_equal(got, hm.kv_words_batch(dig[lo:hi], layer, W)), layer


@pytest.mark.parametrize("mode,ctas", [("kernel", 4), ("kernel", 37), ("copy_engine", 0)])
def test_send_mode_bit_exact_with_unaligned_pages(cuda, mode, ctas):
    torch = cuda
    n = 4096
    p = _prompt(n, 3)
    P, D = _engines(n)
    P.set_send_mode(P.SEND_COPY_ENGINE if mode == "copy_engine" else P.SEND_KERNEL, ctas)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, n)
    prefill(P, 1, p, 0, n)
    # D caches the first 1000 tokens (received earlier), then a second request
    # with the same prefix receives [1000, 4095): its first own page starts
    # at position 1000 (slot 0) while P's position 1000 is slot 8 of a page.
    r0 = D.PrepRecv(5, p[:1001], -1)
    P.direct_send_async(1, (0, 1000), 1, r0.addr, 1)
    P.synchronize()
    assert D.DrainReceiveCompletions() == [5]
    r = D.PrepRecv(10, p, -1)
    assert r.match_len == 1000 and r.addr.token_count == n - 1 - 1000
    plan = P.begin_direct_send(1, (1000, n - 1), 1, r.addr, 2)
    # Layer by layer (the overlap pattern) for the first half, one launch for the rest.
    for layer in range(L // 2):
        P.launch_direct_send_async(plan, (layer, layer + 1), 0)
    P.launch_direct_send_async(plan, (L // 2, L), 0)
    P.synchronize()
    assert D.DrainReceiveCompletions() == [10]
    assert D.GetRecord(10).window["received_writes"] == (n - 1 - 1000) * L
    plan.close()
    _check(torch, D, 10, p, 0, n - 1)
    assert start_generate(D, 10, p, n - 1) == hm.generate(p, 1, L, W)


def test_copy_engine_send_after_producer_event(cuda):
    """Copy-engine sends behind the producer's per-layer event: the copies
    wait for the layer's append (which lands late, behind a sleep)."""
    torch = cuda
    from paper_2412_12488_b200 import BatchEntry

    n = 1024
    p = _prompt(n, 4)
    P, D = _engines(n)
    P.set_send_mode(P.SEND_COPY_ENGINE)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, n)
    fplan = P.BeginForward([BatchEntry(1, (0, n))])
    rows = [torch.randint(-2**62, 2**62, (n, W), dtype=torch.int64, device="cuda")
            for _ in range(4)]
    r = D.PrepRecv(7, p, -1)
    plan = P.begin_direct_send(1, (0, n - 1), 1, r.addr, 1)
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream()
    evs = [torch.cuda.Event() for _ in range(L)]
    for layer in range(L):
        with torch.cuda.stream(cs):
            torch.cuda._sleep(1_000_000)
        P.append_rows_async(fplan, layer, rows[layer % 4].data_ptr(), cs.cuda_stream)
        evs[layer].record(cs)
        P.launch_direct_send_after_async(plan, (layer, layer + 1), evs[layer].cuda_event,
                                         ms.cuda_stream)
    torch.cuda.synchronize()
    P.synchronize()
    assert D.DrainReceiveCompletions() == [7]
    got = torch.empty((n - 1) * W, dtype=torch.int64, device="cuda")
    for layer in range(L):
        D.gather_range_async(7, (0, n - 1), layer, got.data_ptr(), 0)
        torch.cuda.synchronize()
        assert torch.equal(got.view(n - 1, W), rows[layer % 4][:n - 1]), layer
    plan.close()
    fplan.close()


def test_copy_engine_rejects_freed_window(cuda):
    n = 256
    p = _prompt(n, 5)
    P, D = _engines(n)
    P.set_send_mode(P.SEND_COPY_ENGINE)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, n)
    prefill(P, 1, p, 0, n)
    r = D.PrepRecv(7, p, -1)
    plan = P.begin_direct_send(1, (0, n - 1), 1, r.addr, 1)
    D.FreeSequence(7)
    with pytest.raises(SplitserveError) as ei:
        P.launch_direct_send_async(plan, (0, L), 0)
    assert ei.value.code == ErrorCode.UnknownAddress
    r2 = D.PrepRecv(8, p, -1)  # the same pages again: nothing was written into them
    assert D.FillOf(8, 0, 0) == 0
    assert D.GetRecord(8).window["received_writes"] == 0
    plan.close()
    del r2


def test_send_mode_validation(cuda):
    P, _ = _engines(64)
    with pytest.raises(SplitserveError) as ei:
        P.set_send_mode(7)
    assert ei.value.code == ErrorCode.InvalidArgument
    with pytest.raises(SplitserveError):
        P.set_send_mode(P.SEND_KERNEL, -1)
