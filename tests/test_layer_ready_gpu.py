"""Per-layer ready flags on the receiving side: ss_wait_receive_layer_async
orders receiver work after layer l's rows landed while later layers are
still in flight (the sender sleeps between per-layer DirectSends).  A
consumer kernel reading the pool behind each wait sees exactly the sender's
rows; layers that arrive through the host path (ApplyRemoteWrite) count
too."""
import numpy as np
import pytest

from paper_2412_12488_b200 import KVCache

pytestmark = pytest.mark.gpu


class _Dev:
    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": shape,
                                         "typestr": "<i8", "version": 3, "strides": None}


def _prompt(n, seed):
    rng = np.random.Generator(np.random.MT19937(seed))
    return [int(x) for x in rng.integers(0, 256, n)]


@pytest.mark.parametrize("host_layers", [(), (1,)])
def test_receiver_waits_per_layer(cuda, host_layers):
    torch = cuda
    L, W, P = 4, 64, 16
    n = 300
    p = _prompt(n, 3)
    S = KVCache(num_pages=64, page_size=P, layers=L, dim=W, device=0, rank=0)
    D = KVCache(num_pages=64, page_size=P, layers=L, dim=W, device=0, rank=1)
    S.attach_peer(1, D)
    S.CreateSequence(1, p)
    S.EnsureAllocated(1, n)
    rows = torch.randint(-2**62, 2**62, (L, n, W), dtype=torch.int64, device="cuda")
    from paper_2412_12488_b200 import BatchEntry
    plan = S.BeginForward([BatchEntry(1, (0, n))])
    S.append_rows_layers_async(plan, (0, L), rows.data_ptr(), 0)
    torch.cuda.synchronize()
    plan.close()
    r = D.PrepRecv(7, p, -1)
    m, e = r.match_len, r.match_len + r.addr.token_count
    slots = torch.tensor(r.addr.slots(P), dtype=torch.int64, device="cuda")
    # host-path layers first (the transfer agent's frames)
    for layer in host_layers:
        st = D.ApplyRemoteWrite(r.addr, layer, S.GatherRange(1, (m, e), layer), 0)
        assert int(st) == 0
    s_send, s_recv = torch.cuda.Stream(), torch.cuda.Stream()
    # Load the torch kernels used below before any wait spins: with lazy
    # module loading a first-time launch can block until the device idles,
    # which a spinning receiver wait never does before its timeout.  (The
    # library preloads its own kernels when a cache is created.)
    view0 = torch.as_tensor(_Dev(D.pool_layer_ptr(0), (64 * P, W)), device="cuda")
    view0.index_select(0, slots).clone()
    torch.cuda._sleep(1)
    torch.cuda.synchronize()
    dplan = S.begin_direct_send(1, (m, e), 1, r.addr, 3)
    outs = []
    # receiver: per-layer waits then a consumer kernel per layer, queued now
    for layer in range(L):
        D.wait_receive_layer_async(7, layer, 20000, s_recv.cuda_stream)
        view = torch.as_tensor(_Dev(D.pool_layer_ptr(layer), (64 * P, W)), device="cuda")
        with torch.cuda.stream(s_recv):
            outs.append(view.index_select(0, slots).clone())
    # sender: device-direct layers one at a time, ~2 ms apart
    for layer in range(L):
        if layer in host_layers:
            continue
        with torch.cuda.stream(s_send):
            torch.cuda._sleep(4_000_000)
        S.launch_direct_send_async(dplan, (layer, layer + 1), s_send.cuda_stream)
    torch.cuda.synchronize()
    S.synchronize()
    D.synchronize()
    dplan.close()
    for layer in range(L):
        assert torch.equal(outs[layer], rows[layer, m:e]), layer
    assert D.DrainReceiveCompletions() == [7]
