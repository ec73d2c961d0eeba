"""Paged causal GQA prefill attention on tcgen05 (csrc/prefill_attn.cu)
against a plain fp32 PyTorch reference of the same op: queries at positions
[q_begin, q_end) of one sequence attend to keys [0, pos], read through the
sequence's device page table (fragmented pages).  Tolerance as for decode:

    max |out - ref| <= 2e-2   and   rms(out - ref) / rms(ref) <= 2e-2

(bf16 in/out; fp32 accumulation in TMEM; softmax weights rounded to bf16 for
the PV product)."""
import pytest

from paper_2412_12488_b200 import BatchEntry, ErrorCode, KVCache, SplitserveError

pytestmark = pytest.mark.gpu


def _setup(torch, hkv, hd, n, layers=2, P=16, seed=0):
    W = 4 * hkv * hd // 8
    pages = (n + P - 1) // P + 8
    c = KVCache(num_pages=pages + 40, page_size=P, layers=layers, dim=W, device=0)
    for i in range(40):  # fragment the free list
        c.CreateSequence(1000 + i, [i % 7] * P)
        c.EnsureAllocated(1000 + i, P)
    for i in range(0, 40, 2):
        c.FreeSequence(1000 + i)
    c.CreateSequence(1, [i % 13 for i in range(n)])
    c.EnsureAllocated(1, n)
    g = torch.Generator(device="cuda").manual_seed(seed)
    plan = c.BeginForward([BatchEntry(1, (0, n))])
    kv = []
    for layer in range(layers):
        rows = (torch.randn(n, 2, hkv, hd, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
        c.append_rows_async(plan, layer, rows.data_ptr(), 0)
        kv.append((rows[:, 0].float(), rows[:, 1].float()))
    torch.cuda.synchronize()
    plan.close()
    return c, kv


def _ref(torch, q, K, V, q_begin, scale):
    # q [nq, Hq, D]; K/V [n, Hkv, D]; causal: query i (pos q_begin+i) sees keys <= pos.
    nq, hq, _ = q.shape
    n, hkv, _ = K.shape
    Kx = K.repeat_interleave(hq // hkv, dim=1)
    Vx = V.repeat_interleave(hq // hkv, dim=1)
    s = torch.einsum("qhd,nhd->hqn", q.float(), Kx) * scale
    pos = torch.arange(q_begin, q_begin + nq, device=q.device)[:, None]
    keys = torch.arange(n, device=q.device)[None, :]
    s = s.masked_fill((keys > pos)[None], float("-inf"))
    p = torch.softmax(s, dim=-1)
    return torch.einsum("hqn,nhd->qhd", p, Vx)


CASES = [  # (Hq, Hkv, n, q_begin)
    (64, 8, 300, 0),       # full prompt, ragged last tile
    (64, 8, 1000, 800),    # balanced-PD tail (r = 0.2)
    (32, 4, 700, 683),     # 17 queries: partial query block
    (64, 8, 129, 128),     # one query, two key tiles
    (64, 8, 2048, 1536),   # tiles fully inside the causal bound
    (32, 8, 1000, 700),    # Llama 8B heads (G = 4: 32 tokens per tile)
    (32, 8, 4096, 3277),   # Llama 8B balanced-PD tail of a 4K prompt
    (16, 8, 600, 100),     # G = 2 (64 tokens per tile)
    (8, 8, 500, 0),        # MHA (G = 1: 128 tokens per tile)
    (64, 4, 400, 250),     # G = 16 (8 tokens per tile)
]


@pytest.mark.parametrize("case", CASES)
def test_prefill_matches_fp32_reference(cuda, case):
    torch = cuda
    hq, hkv, n, qb = case
    hd = 128
    c, kv = _setup(torch, hkv, hd, n, seed=n)
    g = torch.Generator(device="cuda").manual_seed(qb + 1)
    q = (torch.randn(n - qb, hq, hd, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    out = torch.full_like(q, float("nan"))
    scale = hd ** -0.5
    for layer in range(len(kv)):
        c.paged_prefill_attention_async(1, (qb, n), layer, hq, hkv, hd, scale, q.data_ptr(),
                                        out.data_ptr(), 0)
        torch.cuda.synchronize()
        K, V = kv[layer]
        ref = _ref(torch, q, K, V, qb, scale)
        err = (out.float() - ref).abs()
        assert err.max().item() <= 2e-2, (case, layer, err.max().item())
        rel = (out.float() - ref).pow(2).mean().sqrt() / ref.pow(2).mean().sqrt()
        assert rel.item() <= 2e-2, (case, layer, rel.item())


@pytest.mark.parametrize("page_size", [8, 32, 64, 128, 256])
def test_prefill_page_sizes(cuda, page_size):
    torch = cuda
    hq, hkv, hd, n, qb = 64, 8, 128, 777, 500
    c, kv = _setup(torch, hkv, hd, n, layers=1, P=page_size, seed=page_size)
    q = (torch.randn(n - qb, hq, hd, device="cuda") * 0.5).to(torch.bfloat16)
    out = torch.empty_like(q)
    c.paged_prefill_attention_async(1, (qb, n), 0, hq, hkv, hd, hd ** -0.5, q.data_ptr(),
                                    out.data_ptr(), 0)
    torch.cuda.synchronize()
    ref = _ref(torch, q, kv[0][0], kv[0][1], qb, hd ** -0.5)
    assert (out.float() - ref).abs().max().item() <= 2e-2


@pytest.mark.parametrize("fork_len", [37, 64, 129])
def test_prefill_over_forked_sequence(cuda, fork_len):
    """A child forked at a non-page-aligned length reads [0, fork_len) through
    the parent's pages and the rest through its own, so position chunks are
    not one contiguous page: the per-row load path."""
    torch = cuda
    hq, hkv, hd, P = 64, 8, 128, 16
    n_parent, n = 300, 700
    W = 4 * hkv * hd // 8
    c = KVCache(num_pages=128, page_size=P, layers=1, dim=W, device=0)
    toks = [i % 13 for i in range(n)]
    c.CreateSequence(1, toks[:n_parent])
    c.EnsureAllocated(1, n_parent)
    rows_p = (torch.randn(n_parent, 2, hkv, hd, device="cuda") * 0.5).to(torch.bfloat16)
    plan = c.BeginForward([BatchEntry(1, (0, n_parent))])
    c.append_rows_async(plan, 0, rows_p.data_ptr(), 0)
    torch.cuda.synchronize()
    plan.close()
    c.ForkSequence(1, 2, fork_len, toks)
    c.EnsureAllocated(2, n)
    rows_c = (torch.randn(n - fork_len, 2, hkv, hd, device="cuda") * 0.5).to(torch.bfloat16)
    plan = c.BeginForward([BatchEntry(2, (fork_len, n))])
    c.append_rows_async(plan, 0, rows_c.data_ptr(), 0)
    torch.cuda.synchronize()
    plan.close()
    K = torch.cat([rows_p[:fork_len, 0], rows_c[:, 0]]).float()
    V = torch.cat([rows_p[:fork_len, 1], rows_c[:, 1]]).float()
    qb = 5
    q = (torch.randn(n - qb, hq, hd, device="cuda") * 0.5).to(torch.bfloat16)
    out = torch.empty_like(q)
    c.paged_prefill_attention_async(2, (qb, n), 0, hq, hkv, hd, hd ** -0.5, q.data_ptr(),
                                    out.data_ptr(), 0)
    torch.cuda.synchronize()
    ref = _ref(torch, q, K, V, qb, hd ** -0.5)
    err = (out.float() - ref).abs()
    assert err.max().item() <= 2e-2, err.max().item()


def test_prefill_last_query_equals_decode(cuda):
    """The last query row of a prefill is a decode step over the same context."""
    torch = cuda
    hq, hkv, hd, n = 64, 8, 128, 777
    c, _ = _setup(torch, hkv, hd, n, layers=1)
    q = (torch.randn(1, hq, hd, device="cuda") * 0.5).to(torch.bfloat16)
    a = torch.empty_like(q)
    b = torch.empty_like(q)
    c.paged_prefill_attention_async(1, (n - 1, n), 0, hq, hkv, hd, hd ** -0.5, q.data_ptr(),
                                    a.data_ptr(), 0)
    d = c.begin_decode([1], [n])
    c.paged_decode_attention_async(d, 0, hq, hkv, hd, hd ** -0.5, q.data_ptr(), b.data_ptr(), 0)
    torch.cuda.synchronize()
    assert (a.float() - b.float()).abs().max().item() <= 1e-2
    d.close()


def test_prefill_rejects_bad_arguments(cuda):
    torch = cuda
    c, _ = _setup(torch, 8, 128, 40, layers=1)
    q = torch.zeros(8, 64, 128, dtype=torch.bfloat16, device="cuda")
    # (a group of 3 query heads per KV head does not divide a 128-row tile)
    for args in [((30, 50), 0, 64, 8), ((10, 10), 0, 64, 8), ((0, 8), 1, 64, 8),
                 ((0, 8), 0, 24, 8)]:
        with pytest.raises(SplitserveError) as ei:
            c.paged_prefill_attention_async(1, args[0], args[1], args[2], args[3], 128, 0.1,
                                            q.data_ptr(), q.data_ptr(), 0)
        assert ei.value.code == ErrorCode.InvalidArgument
    with pytest.raises(SplitserveError):
        c.paged_prefill_attention_async(99, (0, 8), 0, 64, 8, 128, 0.1, q.data_ptr(),
                                        q.data_ptr(), 0)
