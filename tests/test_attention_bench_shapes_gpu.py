"""Attention parity at the exact shapes bench.py reports (Llama-3.1-70B
heads: Hq = 64, Hkv = 8, D = 128, page 16), against fp32 PyTorch
references computed in chunks on the GPU.  Same tolerance as the small-shape
tests, written here once:

    max |out - ref| <= 2e-2   and   rms(out - ref) / rms(ref) <= 2e-2

Decode: batch {1, 8, 32, 128} x context {4K, 8K, 32K} — where the stream-K
split cuts a segment into up to 32 pieces — with the split pieces merged by
the separate combine kernel, by the attention kernel's last-arriving CTA,
and by the automatic choice (MICROKV_DECODE_COMBINE), pages fragmented by
the LIFO allocator for batches up to 32.  Prefill: the balanced-PD tail
[6554, 8192) of an 8K prompt and a full 8K causal prefill."""
import numpy as np
import pytest

from paper_2412_12488_b200 import BatchEntry, KVCache

pytestmark = pytest.mark.gpu

HQ, HKV, HD, PAGE = 64, 8, 128, 16
W = 4 * HKV * HD // 8
TOL = 2e-2


def _check(torch, out, ref, what):
    err = (out.float() - ref).abs().max().item()
    rel = ((out.float() - ref).pow(2).mean().sqrt() / ref.pow(2).mean().sqrt()).item()
    assert err <= TOL and rel <= TOL, (what, err, rel)
    return err, rel


def _cache_with_rows(torch, batch, ctx, frag, seed):
    pages = batch * (ctx // PAGE) + 8
    c = KVCache(num_pages=pages + (64 if frag else 0), page_size=PAGE, layers=1, dim=W, device=0)
    if frag:  # every page handed out, then freed in random order: LIFO reuse scatters them
        rng = np.random.default_rng(seed)
        n_all = pages + 64
        per = max(1, n_all // 4096)  # pages per filler sequence (bounded sequence count)
        n_seq = n_all // per
        for i in range(n_seq):
            c.CreateSequence(10**6 + i, [0] * (PAGE * per))
            c.EnsureAllocated(10**6 + i, PAGE * per)
        for i in rng.permutation(n_seq):
            c.FreeSequence(10**6 + int(i))
    for b in range(batch):
        c.CreateSequence(b, [b % 256] * ctx)
        c.EnsureAllocated(b, ctx)
    g = torch.Generator(device="cuda").manual_seed(seed)
    rows = (torch.randn(batch * ctx, 2, HKV, HD, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    plan = c.BeginForward([BatchEntry(b, (0, ctx)) for b in range(batch)])
    c.append_rows_async(plan, 0, rows.data_ptr(), 0)
    torch.cuda.synchronize()
    plan.close()
    return c, rows


def _decode_ref(torch, q, rows, b, ctx, scale):
    K = rows[b * ctx:(b + 1) * ctx, 0].float()  # [n, Hkv, D]
    V = rows[b * ctx:(b + 1) * ctx, 1].float()
    qg = q[b].float().view(HKV, HQ // HKV, HD)   # [Hkv, G, D]
    s = torch.einsum("hgd,nhd->hgn", qg, K) * scale
    return torch.einsum("hgn,nhd->hgd", torch.softmax(s, -1), V).reshape(HQ, HD)


@pytest.mark.parametrize("batch,ctx", [(b, c) for b in (1, 8, 32, 128) for c in (4096, 8192, 32768)])
def test_decode_bench_shapes(cuda, batch, ctx, monkeypatch):
    torch = cuda
    frag = batch in (1, 8, 32) and not (batch == 32 and ctx == 32768)
    c, rows = _cache_with_rows(torch, batch, ctx, frag, seed=batch * 7 + ctx)
    plan = c.begin_decode(list(range(batch)), [ctx] * batch)
    g = torch.Generator(device="cuda").manual_seed(ctx + batch)
    q = (torch.randn(batch, HQ, HD, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    scale = HD ** -0.5
    refs = [_decode_ref(torch, q, rows, b, ctx, scale) for b in range(batch)]
    # The default (TMA page-chunk kernel), then k_decode_attn with each merge.
    for combine in ("auto", "kernel", "fused"):
        if combine == "auto":
            monkeypatch.delenv("MICROKV_DECODE_COMBINE", raising=False)
            monkeypatch.delenv("MICROKV_DECODE_KERNEL", raising=False)
        else:
            monkeypatch.setenv("MICROKV_DECODE_KERNEL", "v1")
            monkeypatch.setenv("MICROKV_DECODE_COMBINE", combine)
        out = torch.full_like(q, float("nan"))
        c.paged_decode_attention_async(plan, 0, HQ, HKV, HD, scale, q.data_ptr(), out.data_ptr(), 0)
        torch.cuda.synchronize()
        for b in range(batch):
            _check(torch, out[b], refs[b], (batch, ctx, combine, b))
    plan.close()


def _prefill_ref(torch, q, K, V, q_begin, scale, head_chunk=8):
    nq = q.shape[0]
    n = K.shape[0]
    out = torch.empty(nq, HQ, HD, device=q.device)
    pos = torch.arange(q_begin, q_begin + nq, device=q.device)[:, None]
    mask = torch.arange(n, device=q.device)[None, :] > pos  # [nq, n]
    for h0 in range(0, HQ, head_chunk):
        hs = range(h0, h0 + head_chunk)
        kv = [h // (HQ // HKV) for h in hs]
        Kh = K[:, kv].float()  # [n, hc, D]
        Vh = V[:, kv].float()
        s = torch.einsum("qhd,nhd->hqn", q[:, h0:h0 + head_chunk].float(), Kh) * scale
        s = s.masked_fill(mask[None], float("-inf"))
        out[:, h0:h0 + head_chunk] = torch.einsum("hqn,nhd->qhd", torch.softmax(s, -1), Vh)
    return out


@pytest.mark.parametrize("q_begin", [6554, 0])
def test_prefill_bench_shapes(cuda, q_begin):
    torch = cuda
    n = 8192
    c, rows = _cache_with_rows(torch, 1, n, frag=True, seed=q_begin + 3)
    g = torch.Generator(device="cuda").manual_seed(q_begin + 11)
    q = (torch.randn(n - q_begin, HQ, HD, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    out = torch.full_like(q, float("nan"))
    scale = HD ** -0.5
    c.paged_prefill_attention_async(0, (q_begin, n), 0, HQ, HKV, HD, scale, q.data_ptr(),
                                    out.data_ptr(), 0)
    torch.cuda.synchronize()
    ref = _prefill_ref(torch, q, rows[:, 0], rows[:, 1], q_begin, scale)
    _check(torch, out, ref, ("prefill", q_begin))
