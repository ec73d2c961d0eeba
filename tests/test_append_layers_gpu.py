"""KV append of several layers in one launch (ss_append_rows_layers_async):
bit-exact against per-layer appends, same write rule (Empty slots only,
kv_cache.cc:328-334: a second append over written slots changes nothing),
same fill states."""
import numpy as np
import pytest

from paper_2412_12488_b200 import BatchEntry, FillState, KVCache

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("W,n,layers", [(512, 300, 6), (128, 1000, 4), (8, 77, 3)])
def test_layers_append_matches_per_layer(cuda, W, n, layers):
    torch = cuda
    mk = lambda: KVCache(num_pages=(n + 15) // 16 + 8, page_size=16, layers=layers, dim=W,
                         device=0)
    A, B = mk(), mk()
    rows = torch.randint(-2**62, 2**62, (layers, n, W), dtype=torch.int64, device="cuda")
    rows2 = torch.randint(-2**62, 2**62, (layers, n, W), dtype=torch.int64, device="cuda")
    plans = []
    for E in (A, B):
        E.CreateSequence(1, list(range(n)))
        E.EnsureAllocated(1, n)
        plans.append(E.BeginForward([BatchEntry(1, (0, n))]))
    A.append_rows_layers_async(plans[0], (0, layers), rows.data_ptr(), 0)
    A.append_rows_layers_async(plans[0], (0, layers), rows2.data_ptr(), 0)  # no-op: not Empty
    for layer in range(layers):
        B.append_rows_async(plans[1], layer, rows[layer].data_ptr(), 0)
    # a partial layer range in one launch, over already-written slots
    B.append_rows_layers_async(plans[1], (1, layers), rows2[1:].data_ptr(), 0)
    torch.cuda.synchronize()
    for layer in range(layers):
        ga, gb = A.GatherRange(1, (0, n), layer), B.GatherRange(1, (0, n), layer)
        assert np.array_equal(ga, gb), layer
        want = rows[layer].cpu().numpy().reshape(-1).view(np.uint64)
        assert np.array_equal(ga, want), layer
        for pos in (0, n // 2, n - 1):
            assert A.FillOf(1, pos, layer) == B.FillOf(1, pos, layer) == FillState.ComputedLocal
    for p in plans:
        p.close()


def test_layers_append_rejects_bad_range(cuda):
    from paper_2412_12488_b200 import ErrorCode, SplitserveError
    E = KVCache(num_pages=8, page_size=16, layers=3, dim=8, device=0)
    E.CreateSequence(1, list(range(20)))
    E.EnsureAllocated(1, 20)
    p = E.BeginForward([BatchEntry(1, (0, 20))])
    for rng in ((0, 0), (2, 1), (0, 4), (-1, 2)):
        with pytest.raises(SplitserveError) as ei:
            E.append_rows_layers_async(p, rng, 0, 0)
        assert ei.value.code == ErrorCode.InvalidArgument
    p.close()
