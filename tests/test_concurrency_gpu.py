"""The reference's threading contract (kv_cache.h:12-15): one
executor owns every mutating call while the transfer agent applies remote
writes concurrently.  Here a second thread feeds encoded write frames into
a B200 receiver (ReceiveWriteFrame: H2D, CRC on the GPU, ApplyRemoteWrite on
the receive stream) while the executor thread generates on other sequences
and creates / frees sequences; everything stays exact against the oracle."""
import threading
import time

import numpy as np
import pytest

from flows import prefill
from oracle import hashmodel as hm
from paper_2412_12488_b200 import KVCache
from paper_2412_12488_b200.engine import Engine

pytestmark = pytest.mark.gpu
L, W = 4, 64


def _prompt(n, seed):
    rng = np.random.Generator(np.random.MT19937(seed))
    return [int(x) for x in rng.integers(0, 256, n)]


@pytest.mark.parametrize("rounds", [3])
def test_transfer_agent_thread_beside_executor(cuda, rounds):
    for r in range(rounds):
        D = KVCache(num_pages=512, page_size=16, layers=L, dim=W, device=0, rank=1)
        P = KVCache(num_pages=512, page_size=16, layers=L, dim=W, device=0, rank=0)
        a = _prompt(700, 10 + r)
        res = D.PrepRecv(1, a, -1)
        m, e = res.match_len, res.match_len + res.addr.token_count
        P.CreateSequence(20, a)
        P.EnsureAllocated(20, e)
        prefill(P, 20, a, 0, e)
        # several frames per layer (chunks of the address), in shuffled order
        frames = []
        for layer in range(L):
            for lo in range(m, e, 128):
                hi = min(e, lo + 128)
                frames.append(P.EncodeWriteFrame(20, (lo, hi), layer, 7, res.addr.Slice(lo, hi)))
        np.random.default_rng(r).shuffle(frames)
        acks, errors = [], []

        def agent():
            try:
                for f in frames:
                    acks.append(D.ReceiveWriteFrame(f))
                    time.sleep(0.0005)
            except Exception as ex:  # noqa: BLE001
                errors.append(ex)

        t = threading.Thread(target=agent)
        t.start()
        # Executor work on the same receiver meanwhile.
        E = Engine(D, 1)
        outs = []
        for k in range(4):
            p = _prompt(90 + 13 * k, 100 + 10 * r + k)
            outs.append((p, E.api_start_generate(p, 0, 3)))
            D.CreateSequence(500 + k, _prompt(40, k))
            D.EnsureAllocated(500 + k, 40)
            D.FreeSequence(500 + k)
        t.join()
        assert not errors, errors
        assert all(st == 0 for _, st in acks), [st for _, st in acks]
        for p, toks in outs:
            assert toks == hm.generate(p, 3, L, W)
        # The executor's own step loop may already have drained the
        # completion (each completion is handed out once): check the record.
        D.DrainReceiveCompletions()
        rec = D.GetRecord(1)
        assert rec.finished and rec.window and rec.window["complete"] and D.Committed(1) == e
        dig = hm.prefix_digests(a[:e])
        for layer in range(L):
            got = D.GatherRange(1, (0, e), layer).reshape(e, W)
            assert np.array_equal(got, hm.kv_words_batch(dig, layer, W)), layer
