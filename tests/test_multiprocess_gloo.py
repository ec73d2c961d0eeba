"""The N>1 control path on CPU (world_size 2, gloo, 127.0.0.1): the decode
rank reserves pages (prep_recv) and ships the KVAddrInfo to the prefill
rank the way bench.py does at N>1; the prefill rank declares the send and
plans it.  Host-only caches: the bookkeeping is the product's, no device.
The max-over-ranks timing reduction bench.py uses is exercised too."""
import os
import socket
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    try:
        import numpy as np
        import torch
        import torch.distributed as dist

        from oracle.kvcache_oracle import KVCache as OracleCache
        from paper_2412_12488_b200 import BatchEntry, KVCache, SplitserveError

        dist.init_process_group("gloo", rank=rank, world_size=world)
        rng = np.random.Generator(np.random.MT19937(5))
        prompt = [int(x) for x in rng.integers(0, 256, 300)]
        me = KVCache(num_pages=64, page_size=16, layers=4, dim=128, device=-1, rank=rank)
        if rank == 1:  # decode engine
            try:
                me.export_ipc()
                ipc_refused = False
            except SplitserveError as e:
                ipc_refused = e.name == "NoDevice"
            r = me.PrepRecv(10, prompt, -1)
            dist.send_object_list([(r.match_len, r.addr)], dst=0)
            result = ("D", ipc_refused, me.FreePages(), me.GetRecord(10).window)
        else:  # prefill engine
            obj = [None]
            dist.recv_object_list(obj, src=1)
            m, addr = obj[0]
            want = OracleCache(num_pages=64, page_size=16, layers=4, dim=128).PrepRecv(10, prompt, -1)
            me.CreateSequence(20, prompt)
            me.EnsureAllocated(20, 299)
            me.MarkSend(20, (m, 299), 1, addr, 1)
            plan = me.BeginForward([BatchEntry(20, (0, 299))])
            result = ("P", m == want.match_len and addr == want.addr, plan.num_sends,
                      plan.total_outputs, me.PendingSendCount())
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, result, float(t[0])))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as ex:
        q.put((rank, ("error", repr(ex)), None))


def test_two_rank_prep_recv_and_send_plan():
    import torch.multiprocessing as tmp

    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, result, mx = q.get(timeout=120)
        res[rank] = (result, mx)
    for p in procs:
        p.join(30)
    assert res[1][0][0] == "D" and res[1][0][1], res[1]
    assert res[1][0][3]["range"] == (0, 299)
    assert res[0][0] == ("P", True, 1, 299, 0), res[0]
    assert res[0][1] == res[1][1] == 2.0
