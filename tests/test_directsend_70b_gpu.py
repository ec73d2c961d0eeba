"""The headline migration at the bench's exact shape: Llama-3.1-70B KV (80
layers, W=512 words = 4 KiB per token-layer, page 16), an 8,192-token
prompt, D.PrepRecv(end=-1) -> 8,191 tokens, one DirectSend of all 80
layers.  Every received row of every layer is compared with the oracle's
KvEntryWords (hash_model.cc:27-46) and the next token with the oracle's
Generate.  Run once with device-scope publication (P and D on one GPU) and
once with MICROKV_FORCE_SYS_SCOPE=1 (the cross-GPU branch of the copy
kernel: system-scope fence and red.release.sys window counters); and, with
two GPUs visible, P on cuda:0 storing into D on cuda:1 over NVLink."""
import numpy as np
import pytest

from flows import prefill, start_generate

from oracle import hashmodel as hm
from paper_2412_12488_b200 import KVCache

pytestmark = pytest.mark.gpu

L, W, PAGE, N = 80, 512, 16, 8192


def _prompt():
    return np.random.Generator(np.random.MT19937(1)).integers(0, 256, N).astype(np.int32)


def _check_received(torch, D, seq, dig, n, dev):
    out = torch.empty(n * W, dtype=torch.int64, device=f"cuda:{dev}")
    for layer in range(L):
        D.gather_range_async(seq, (0, n), layer, out.data_ptr(), 0)
        torch.cuda.synchronize(dev)
        got = out.cpu().numpy().view(np.uint64).reshape(n, W)
        want = hm.kv_words_batch(dig[:n], layer, W)
        assert np.array_equal(got, want), f"layer {layer}"


@pytest.mark.parametrize("mode", ["device_scope", "force_sys_scope", "two_gpus"])
def test_70b_8k_directsend_all_layers_bit_exact(cuda, mode, monkeypatch):
    torch = cuda
    d_dev = 1 if mode == "two_gpus" else 0
    if mode == "two_gpus" and torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    if mode == "force_sys_scope":
        monkeypatch.setenv("MICROKV_FORCE_SYS_SCOPE", "1")  # read at cache creation
    p = _prompt()
    pages = N // PAGE + 8
    P = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=0)
    D = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=d_dev, rank=1)
    P.attach_peer(1, D)
    assert P.peer_info(1)["sys_scope"] == (mode != "device_scope")
    P.CreateSequence(1, p)
    P.EnsureAllocated(1, N)
    prefill(P, 1, p, 0, N)  # toy-model KV of every (position, layer) in P's pages
    assert P.Committed(1) == N
    r = D.PrepRecv(10, p, -1)
    assert r.match_len == 0 and r.addr.token_count == N - 1
    assert len(r.addr.ranges) == N // PAGE
    plan = P.begin_direct_send(1, (0, N - 1), 1, r.addr, 7)
    P.launch_direct_send_async(plan, (0, L), 0)
    P.synchronize()
    assert D.DrainReceiveCompletions() == [10]
    assert D.GetRecord(10).window["received_writes"] == (N - 1) * L
    plan.close()
    _check_received(torch, D, 10, hm.prefix_digests(p), N - 1, d_dev)
    assert D.Committed(10) == N - 1
    assert start_generate(D, 10, p, N - 1) == hm.generate(p, 1, L, W)
