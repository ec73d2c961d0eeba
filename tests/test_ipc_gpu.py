"""Cross-process remote_send through CUDA IPC: engine D in one process
exports its receive surface; engine P in another imports it and stores KV
straight into D's reserved pages (the multi-GPU path).  D checks the
received rows against the oracle and generates the reference token.

Modes: both processes on cuda:0 (device-scope publication); the same with
MICROKV_FORCE_SYS_SCOPE=1 (the cross-GPU branch: system-scope fence and
red.release.sys counters, runnable on one GPU); D on cuda:1 and P on
cuda:0 (real NVLink peer stores; skipped with fewer than two GPUs)."""
import multiprocessing as mp
import os
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
L, W, N = 4, 512, 1024


def _prompt():
    import numpy as np

    rng = np.random.Generator(np.random.MT19937(31))
    return [int(x) for x in rng.integers(0, 256, N)]


def _decode_proc(q_out, q_in, dev):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    try:
        import numpy as np

        from flows import start_generate
        from oracle import hashmodel as hm
        from paper_2412_12488_b200 import KVCache

        p = _prompt()
        D = KVCache(num_pages=N // 16 + 4, page_size=16, layers=L, dim=W, device=dev, rank=1)
        r = D.PrepRecv(10, p, -1)
        q_out.put(("addr", D.export_ipc(), r.match_len, r.addr))
        assert q_in.get(timeout=120) == "sent"
        done = D.DrainReceiveCompletions()
        assert done == [10], done
        dig = hm.prefix_digests(p)
        for layer in range(L):
            got = D.GatherRange(10, (0, N - 1), layer).reshape(N - 1, W)
            assert np.array_equal(got, hm.kv_words_batch(dig[:N - 1], layer, W)), layer
        tok = start_generate(D, 10, p, N - 1)
        assert tok == hm.generate(p, 1, L, W), tok
        q_out.put(("ok", tok))
    except BaseException as ex:  # report, never hang the parent
        q_out.put(("error", repr(ex)))


def _prefill_proc(q_from_d, q_to_d, q_out, dev, want_sys):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    try:
        from flows import prefill
        from paper_2412_12488_b200 import KVCache

        p = _prompt()
        msg = q_from_d.get(timeout=120)
        assert msg[0] == "addr", msg
        _, handle, m, addr = msg
        P = KVCache(num_pages=N // 16 + 4, page_size=16, layers=L, dim=W, device=dev, rank=0)
        P.import_ipc(1, handle)
        info = P.peer_info(1)
        assert info["sys_scope"] == want_sys, info
        P.CreateSequence(20, p)
        P.EnsureAllocated(20, N - 1)
        P.MarkSend(20, (m, N - 1), 1, addr, 3)
        prefill(P, 20, p, 0, N - 1)
        P.synchronize()
        P.detach_peer(1)
        q_to_d.put("sent")
        q_out.put(("ok",))
    except BaseException as ex:
        q_to_d.put("failed")
        q_out.put(("error", repr(ex)))


@pytest.mark.parametrize("mode", ["same_gpu", "force_sys_scope", "two_gpus"])
def test_remote_send_across_processes(cuda, mode, monkeypatch):
    d_dev, p_dev, want_sys = {"same_gpu": (0, 0, False), "force_sys_scope": (0, 0, True),
                              "two_gpus": (1, 0, True)}[mode]
    if mode == "two_gpus" and cuda.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (P on cuda:0 stores into D on cuda:1 over NVLink)")
    if mode == "force_sys_scope":
        monkeypatch.setenv("MICROKV_FORCE_SYS_SCOPE", "1")  # inherited by the spawned engines
    ctx = mp.get_context("spawn")
    d_out, to_d, p_out, d_to_p = ctx.Queue(), ctx.Queue(), ctx.Queue(), ctx.Queue()
    dp = ctx.Process(target=_decode_proc, args=(d_out, to_d, d_dev))
    dp.start()
    first = d_out.get(timeout=180)
    if first[0] == "error":
        dp.join(10)
        pytest.fail(first[1])
    d_to_p.put(first)
    pp = ctx.Process(target=_prefill_proc, args=(d_to_p, to_d, p_out, p_dev, want_sys))
    pp.start()
    pres = p_out.get(timeout=180)
    dres = d_out.get(timeout=180)
    pp.join(30)
    dp.join(30)
    assert pres[0] == "ok", pres
    assert dres[0] == "ok", dres
