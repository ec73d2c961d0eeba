"""Paged GQA decode attention (bf16 in, fp32 accumulate, bf16 out) against a
plain fp32 PyTorch reference of the same op.  No reference analogue exists
(the reference's attention is the integer fold), so the tolerance is ours:

    max |out - ref| <= 2e-2   and   rms(out - ref) / rms(ref) <= 2e-2

(bf16 output rounding alone is 2^-9 relative; the kernel also rounds the
softmax weights to bf16 before the PV product).  Contexts are ragged and the
pages fragmented (interleaved allocation, then frees and reuse), so every
read goes through the device page table."""
import numpy as np
import pytest

from paper_2412_12488_b200 import BatchEntry, ErrorCode, KVCache, SplitserveError

pytestmark = pytest.mark.gpu

SHAPES = [  # (Hq, Hkv, D) with dim = 4 * Hkv * D / 8 u64 words
    (8, 4, 64),     # tiny config: W = 128
    (32, 8, 128),   # Llama-3.1-8B
    (64, 8, 128),   # Llama-3.1-70B
]


def _fill(torch, cache, seqs_ctx, hkv, hd, layers, page_size, seed):
    """Appends K||V rows for every (seq, pos, layer); returns {seq: [layer] -> (K, V)}."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    kv = {}
    batch = [BatchEntry(s, (0, n)) for s, n in seqs_ctx]
    total = sum(n for _, n in seqs_ctx)
    plan = cache.BeginForward(batch)
    for layer in range(layers):
        rows = (torch.randn(total, 2, hkv, hd, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
        cache.append_rows_async(plan, layer, rows.data_ptr(), 0)
        off = 0
        for s, n in seqs_ctx:
            kv.setdefault(s, []).append((rows[off:off + n, 0].float(), rows[off:off + n, 1].float()))
            off += n
    torch.cuda.synchronize()
    plan.close()
    return kv


def _ref(torch, q, K, V, scale):
    # q [Hq, D], K/V [n, Hkv, D] -> [Hq, D] in fp32.
    hq, hkv = q.shape[0], K.shape[1]
    g = hq // hkv
    Kx = K.repeat_interleave(g, dim=1)  # [n, Hq, D]
    Vx = V.repeat_interleave(g, dim=1)
    s = torch.einsum("hd,nhd->hn", q.float(), Kx) * scale
    p = torch.softmax(s, dim=-1)
    return torch.einsum("hn,nhd->hd", p, Vx)


@pytest.mark.parametrize("combine", ["auto", "v1-kernel", "v1-fused"])
@pytest.mark.parametrize("shape", SHAPES)
def test_decode_matches_fp32_reference(cuda, shape, combine, monkeypatch):
    """The default kernel for the shape (the TMA page-chunk kernel for 8 KV
    heads x 128, decode_pages.cu; k_decode_attn otherwise), and k_decode_attn
    forced (MICROKV_DECODE_KERNEL=v1) with its split segments merged by the
    separate combine kernel or by the attention kernel's last arriving CTA
    (MICROKV_DECODE_COMBINE): same tolerance."""
    if combine != "auto":
        monkeypatch.setenv("MICROKV_DECODE_KERNEL", "v1")
        monkeypatch.setenv("MICROKV_DECODE_COMBINE", combine.split("-")[1])
    torch = cuda
    hq, hkv, hd = shape
    W = 4 * hkv * hd // 8
    P, layers = 16, 2
    ctx = [1, 15, 16, 17, 300, 1000, 2048]
    c = KVCache(num_pages=600, page_size=P, layers=layers, dim=W, device=0)
    # Fragment the free list: interleave short allocations, free every other one.
    for i in range(40):
        c.CreateSequence(1000 + i, [i % 7] * 40)
        c.EnsureAllocated(1000 + i, 40)
    for i in range(0, 40, 2):
        c.FreeSequence(1000 + i)
    seqs = []
    for b, n in enumerate(ctx):
        c.CreateSequence(b, [(b + i) % 11 for i in range(n)])
        c.EnsureAllocated(b, n)
        seqs.append((b, n))
    kv = _fill(torch, c, seqs, hkv, hd, layers, P, seed=hq)
    plan = c.begin_decode([s for s, _ in seqs], [n for _, n in seqs])
    scale = hd ** -0.5
    q = (torch.randn(len(seqs), hq, hd, device="cuda") * 0.5).to(torch.bfloat16)
    out = torch.empty_like(q)
    for layer in range(layers):
        c.paged_decode_attention_async(plan, layer, hq, hkv, hd, scale, q.data_ptr(),
                                       out.data_ptr(), 0)
        torch.cuda.synchronize()
        for b, (s, n) in enumerate(seqs):
            K, V = kv[s][layer]
            ref = _ref(torch, q[b], K, V, scale)
            err = (out[b].float() - ref).abs()
            assert err.max().item() <= 2e-2, (shape, n, layer, err.max().item())
            rel = (out[b].float() - ref).pow(2).mean().sqrt() / ref.pow(2).mean().sqrt()
            assert rel.item() <= 2e-2, (shape, n, layer, rel.item())
    plan.close()


@pytest.mark.parametrize("kernel", ["auto", "v1"])
@pytest.mark.parametrize("page_size", [1, 4, 8, 32, 64])
def test_decode_page_sizes(cuda, page_size, kernel, monkeypatch):
    """Page sizes other than 16 at the 70B heads: the page-chunk kernel's
    chunks are runs of consecutive slots capped at 16 rows, so pages of 1-8
    slots give chunks shorter than the TMA box (the V-tail zeroing path)
    unless neighbouring pages happen to be adjacent, and pages of 32/64 split
    into full chunks; k_decode_attn (v1) reads through the page table at
    any page size.  Fragmented free list, ragged contexts, fp32 reference."""
    if kernel == "v1":
        monkeypatch.setenv("MICROKV_DECODE_KERNEL", "v1")
    torch = cuda
    hq, hkv, hd = 64, 8, 128
    W = 4 * hkv * hd // 8
    P, layers = page_size, 1
    ctx = [1, 3, 15, 16, 17, 33, 129, 700]
    c = KVCache(num_pages=4096 // P, page_size=P, layers=layers, dim=W, device=0)
    for i in range(24):
        c.CreateSequence(1000 + i, [i % 5] * 24)
        c.EnsureAllocated(1000 + i, 24)
    for i in range(0, 24, 2):
        c.FreeSequence(1000 + i)
    seqs = []
    for b, n in enumerate(ctx):
        c.CreateSequence(b, [(b + 3 * i) % 13 for i in range(n)])
        c.EnsureAllocated(b, n)
        seqs.append((b, n))
    kv = _fill(torch, c, seqs, hkv, hd, layers, P, seed=P)
    plan = c.begin_decode([s for s, _ in seqs], [n for _, n in seqs])
    scale = hd ** -0.5
    g = torch.Generator(device="cuda").manual_seed(100 + P)
    q = (torch.randn(len(seqs), hq, hd, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    out = torch.empty_like(q)
    c.paged_decode_attention_async(plan, 0, hq, hkv, hd, scale, q.data_ptr(), out.data_ptr(), 0)
    torch.cuda.synchronize()
    for b, (s, n) in enumerate(seqs):
        K, V = kv[s][0]
        ref = _ref(torch, q[b], K, V, scale)
        err = (out[b].float() - ref).abs()
        assert err.max().item() <= 2e-2, (P, kernel, n, err.max().item())
        rel = (out[b].float() - ref).pow(2).mean().sqrt() / ref.pow(2).mean().sqrt()
        assert rel.item() <= 2e-2, (P, kernel, n, rel.item())
    plan.close()


def test_decode_rejects_bad_geometry_and_missing_kv(cuda):
    c = KVCache(num_pages=16, page_size=16, layers=1, dim=512, device=0)
    c.CreateSequence(1, [1] * 20)
    c.EnsureAllocated(1, 20)
    with pytest.raises(SplitserveError) as ei:
        c.begin_decode([1], [20])  # no KV appended yet: fill-state safety
    assert ei.value.code == ErrorCode.MissingKV
    torch = cuda
    plan = c.BeginForward([BatchEntry(1, (0, 20))])
    rows = torch.zeros(20 * 4096 // 2, dtype=torch.bfloat16, device="cuda")
    c.append_rows_async(plan, 0, rows.data_ptr(), 0)
    torch.cuda.synchronize()
    d = c.begin_decode([1], [20])
    q = torch.zeros(1, 64, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(SplitserveError) as ei:  # 4*Hkv*D bytes must equal the entry width
        c.paged_decode_attention_async(d, 0, 64, 4, 128, 0.1, q.data_ptr(), q.data_ptr(), 0)
    assert ei.value.code == ErrorCode.InvalidArgument


@pytest.mark.parametrize("kernel", ["auto", "v1"])
def test_decode_over_forked_contexts(cuda, kernel, monkeypatch):
    """Contexts that share a parent's pages (ForkSequence at a position inside
    a page, kv_cache.cc:120-166): the child's positions [0, 21) live in the
    parent's first two pages and [21, n) start at slot 0 of the child's own
    pages (fork-relative paging), so the decode kernels see runs of
    consecutive slots that end mid-page.  Both kernels, fp32 reference."""
    if kernel == "v1":
        monkeypatch.setenv("MICROKV_DECODE_KERNEL", "v1")
    torch = cuda
    hq, hkv, hd = 64, 8, 128
    W = 4 * hkv * hd // 8
    c = KVCache(num_pages=200, page_size=16, layers=1, dim=W, device=0)
    g = torch.Generator(device="cuda").manual_seed(5)
    parent = [(7 * i) % 251 for i in range(37)]
    c.CreateSequence(1, parent)
    c.EnsureAllocated(1, 37)
    pr = (torch.randn(37, 2, hkv, hd, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    plan = c.BeginForward([BatchEntry(1, (0, 37))])
    c.append_rows_async(plan, 0, pr.data_ptr(), 0)
    torch.cuda.synchronize()
    plan.close()
    kv = {1: (pr[:, 0].float(), pr[:, 1].float())}
    for child, fork, n in ((2, 21, 300), (3, 5, 40), (4, 37, 37 + 16 * 3 + 1)):
        toks = parent[:fork] + [(3 * i + child) % 251 for i in range(n - fork)]
        c.ForkSequence(1, child, fork, toks)
        c.EnsureAllocated(child, n)
        rows = (torch.randn(n - fork, 2, hkv, hd, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
        plan = c.BeginForward([BatchEntry(child, (fork, n))])
        c.append_rows_async(plan, 0, rows.data_ptr(), 0)
        torch.cuda.synchronize()
        plan.close()
        kv[child] = (torch.cat([pr[:fork, 0].float(), rows[:, 0].float()]),
                     torch.cat([pr[:fork, 1].float(), rows[:, 1].float()]))
    seqs = [1, 2, 3, 4]
    lens = [kv[s][0].shape[0] for s in seqs]
    dplan = c.begin_decode(seqs, lens)
    q = (torch.randn(len(seqs), hq, hd, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    out = torch.empty_like(q)
    scale = hd ** -0.5
    c.paged_decode_attention_async(dplan, 0, hq, hkv, hd, scale, q.data_ptr(), out.data_ptr(), 0)
    torch.cuda.synchronize()
    for b, s in enumerate(seqs):
        ref = _ref(torch, q[b], kv[s][0], kv[s][1], scale)
        err = (out[b].float() - ref).abs()
        assert err.max().item() <= 2e-2, (kernel, s, err.max().item())
        rel = (out[b].float() - ref).pow(2).mean().sqrt() / ref.pow(2).mean().sqrt()
        assert rel.item() <= 2e-2, (kernel, s, rel.item())
    dplan.close()
