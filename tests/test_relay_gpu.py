"""Relay-chain prefix migration (config 4): an owner's
cached prefix reaches k engines as owner -> T1 -> T2 -> T3, each target
forwarding layer l as soon as layer l has landed in its own pages (device
wait on its per-layer receive counter).  Every target's pages must equal
the oracle's KvEntryWords, windows complete and the last target generates
the oracle's token; a relay whose upstream never sends times out without
forwarding anything.  (All engines share one GPU here; across GPUs each hop
is a separate NVLink link, so the owner's egress carries the prefix once.)"""
import numpy as np
import pytest

from flows import prefill, start_generate

from oracle import hashmodel as hm
from paper_2412_12488_b200 import ErrorCode, KVCache, SplitserveError

pytestmark = pytest.mark.gpu

L, W, PAGE = 8, 512, 16


def _prompt(n, seed):
    return np.random.Generator(np.random.MT19937(seed)).integers(0, 256, n).astype(np.int32)


@pytest.mark.parametrize("owner_layers_per_launch", [1, L])
def test_relay_chain_three_targets(cuda, owner_layers_per_launch):
    torch = cuda
    n, k = 2048, 3
    p = _prompt(n + 1, 11)
    pages = n // PAGE + 8
    O = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=0)
    T = [KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=i + 1)
         for i in range(k)]
    O.attach_peer(1, T[0])
    for i in range(k - 1):
        T[i].attach_peer(i + 2, T[i + 1])
    O.CreateSequence(1, p)
    O.EnsureAllocated(1, n)
    prefill(O, 1, p, 0, n)
    addrs = [t.PrepRecv(10 + i, p, n).addr for i, t in enumerate(T)]  # prep_recv(end=len)
    assert all(a.token_count == n for a in addrs)
    streams = [torch.cuda.Stream() for _ in range(k + 1)]
    # Every kernel launched while relay warps wait must already be loaded:
    # a lazy module load waits for the device to idle (torch's sleep kernel
    # is loaded here, before any relay spins).
    torch.cuda._sleep(1)
    torch.cuda.synchronize()
    # Downstream hops first: each waits on its own receive counters.
    plans = []
    for i in reversed(range(k - 1)):
        pl = T[i].begin_direct_send(10 + i, (0, n), i + 2, addrs[i + 1], 5)
        T[i].launch_relay_send_async(pl, (0, L), 20000, streams[i + 1].cuda_stream)
        plans.append(pl)
    op = O.begin_direct_send(1, (0, n), 1, addrs[0], 5)
    with torch.cuda.stream(streams[0]):
        torch.cuda._sleep(2_000_000)  # the relays are waiting before the first byte leaves
    for lb in range(0, L, owner_layers_per_launch):
        O.launch_direct_send_async(op, (lb, lb + owner_layers_per_launch), streams[0].cuda_stream)
    torch.cuda.synchronize()
    for e in [O] + T:
        e.synchronize()
    dig = hm.prefix_digests(p)
    out = torch.empty(n * W, dtype=torch.int64, device="cuda")
    for i, t in enumerate(T):
        assert t.DrainReceiveCompletions() == [10 + i], i
        assert t.GetRecord(10 + i).window["received_writes"] == n * L
        for layer in range(L):
            t.gather_range_async(10 + i, (0, n), layer, out.data_ptr(), 0)
            torch.cuda.synchronize()
            got = out.cpu().numpy().view(np.uint64).reshape(n, W)
            assert np.array_equal(got, hm.kv_words_batch(dig[:n], layer, W)), (i, layer)
    # The last target serves the request from the migrated prefix.
    assert start_generate(T[-1], 10 + k - 1, p, n) == hm.generate(p, 1, L, W)
    for pl in plans + [op]:
        pl.close()


def test_relay_without_upstream_times_out_and_forwards_nothing(cuda):
    torch = cuda
    n = 256
    p = _prompt(n, 12)
    T1 = KVCache(num_pages=32, page_size=PAGE, layers=2, dim=W, device=0, rank=1)
    T2 = KVCache(num_pages=32, page_size=PAGE, layers=2, dim=W, device=0, rank=2)
    T1.attach_peer(2, T2)
    a1 = T1.PrepRecv(10, p, n).addr
    a2 = T2.PrepRecv(20, p, n).addr
    pl = T1.begin_direct_send(10, (0, n), 2, a2, 1)
    T1.launch_relay_send_async(pl, (0, 2), 50, 0)
    torch.cuda.synchronize()
    with pytest.raises(SplitserveError) as ei:
        T1.synchronize()
    assert ei.value.code == ErrorCode.Aborted
    assert T2.DrainReceiveCompletions() == []
    assert T2.GetRecord(20).window["received_writes"] == 0
    assert T2.FillOf(20, 0, 0) == 0 and T2.FillOf(20, n - 1, 1) == 0
    pl.close()
    del a1
