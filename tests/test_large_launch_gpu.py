"""The largest launch shapes, where the row copies run on a grid of 11 CTAs
per SM (>= 96K items, kernels.cu kHugeItems; profiles/r02/copy_grid_ab.txt):
an 8192-token x 80-layer prefix (70B KV shape, 2.7 GB) appended in one
launch, fanned out to three engines in one launch (k_copy_rows_fanout), and
sent by one 80-layer DirectSend into a fourth; every target's rows, gathered
back in one launch, equal the source rows bit for bit and every receive
window completes with n x L writes (kv_cache.cc:373-387,
kv_cache.cc:409-463)."""
import numpy as np
import pytest

from paper_2412_12488_b200 import BatchEntry, KVCache

pytestmark = pytest.mark.gpu


def test_prefix_fanout_and_directsend_at_70b_8k(cuda):
    torch = cuda
    L, W, n = 80, 512, 8192
    p = np.random.Generator(np.random.MT19937(71)).integers(0, 256, n).astype(np.int32)
    pages = n // 16 + 8
    P = KVCache(num_pages=pages, page_size=16, layers=L, dim=W, device=0, rank=0)
    Ds = [KVCache(num_pages=pages, page_size=16, layers=L, dim=W, device=0, rank=r)
          for r in (1, 2, 3, 4)]
    for D in Ds:
        P.attach_peer(D.rank, D)
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, n)
    plan = P.BeginForward([BatchEntry(1, (0, n))])
    g = torch.Generator(device="cuda").manual_seed(71)
    rows = torch.randint(-2**62, 2**62, (L, n * W), dtype=torch.int64, device="cuda", generator=g)
    P.append_rows_layers_async(plan, (0, L), rows.data_ptr(), 0)
    torch.cuda.synchronize()
    plan.close()
    s = torch.cuda.Stream()
    addrs = [D.PrepRecv(10 + D.rank, p, n).addr for D in Ds]
    P.broadcast_send_async(1, (0, n), [1, 2, 3], addrs[:3], 5, None, s.cuda_stream)
    dplan = P.begin_direct_send(1, (0, n), 4, addrs[3], 6)
    P.launch_direct_send_async(dplan, (0, L), s.cuda_stream)
    s.synchronize()
    P.synchronize()
    dplan.close()
    out = torch.empty_like(rows)
    for D in Ds:
        assert D.DrainReceiveCompletions() == [10 + D.rank]
        assert D.GetRecord(10 + D.rank).window["received_writes"] == n * L
        out.zero_()
        D.gather_range_layers_async(10 + D.rank, (0, n), (0, L), out.data_ptr(), 0)
        torch.cuda.synchronize()
        assert torch.equal(out, rows), D.rank
    del rows, out
    torch.cuda.empty_cache()
