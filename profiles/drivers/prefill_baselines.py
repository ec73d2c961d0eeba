"""Profiling driver: the paged tcgen05 prefill (k_prefill_attn_k128) beside
library attention on the identical math (70B heads Hq=64 Hkv=8 D=128, bf16,
causal with queries at the END of the keys = bottom-right alignment):
  ours          paged, reading K/V through the page table (the product path)
  flash_attn    flash_attn_func(causal=True) on contiguous K/V (bottom-right
                since 2.1)
  sdpa_cudnn /  torch SDPA with causal_lower_right on contiguous K/V, the
  sdpa_flash    cuDNN / flash backends forced
  flashinfer    single_prefill_with_kv_cache(causal=True) on contiguous K/V
Device time per call, 10 calls behind a sleep; TFLOP/s = 4*D*Hq*sum(pos+1)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_12488_b200 import BatchEntry, KVCache  # noqa: E402

HQ, HKV, HD, PAGE, W = 64, 8, 128, 16, 512
try:
    PEAK = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops"])
except Exception:
    PEAK = 2250.0


def dev_time(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(20_000_000)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


res = {}
for ctx, qb in ((8192, 6554), (8192, 0), (32768, 26214)):
    nq = ctx - qb
    c = KVCache(num_pages=ctx // PAGE + 16, page_size=PAGE, layers=1, dim=W, device=0)
    c.CreateSequence(1, np.zeros(ctx, np.int32))
    c.EnsureAllocated(1, ctx)
    plan = c.BeginForward([BatchEntry(1, (0, ctx))])
    rows = (torch.randn(ctx, 2, HKV, HD, device="cuda") * 0.5).to(torch.bfloat16)
    c.append_rows_async(plan, 0, rows.data_ptr(), 0)
    torch.cuda.synchronize()
    plan.close()
    q = (torch.randn(nq, HQ, HD, device="cuda") * 0.5).to(torch.bfloat16)
    o = torch.empty_like(q)
    K = rows[:, 0].contiguous()  # [ctx, Hkv, D]
    V = rows[:, 1].contiguous()
    flops = 4.0 * HD * HQ * sum(range(qb + 1, ctx + 1))
    key = f"q[{qb},{ctx})"
    out = {}
    stream = torch.cuda.current_stream().cuda_stream
    fns = {"ours_paged": lambda: c.paged_prefill_attention_async(
        1, (qb, ctx), 0, HQ, HKV, HD, HD ** -0.5, q.data_ptr(), o.data_ptr(), stream)}
    try:
        from flash_attn import flash_attn_func

        qq, kk, vv = q[None], K[None], V[None]
        fns["flash_attn_2"] = lambda: flash_attn_func(qq, kk, vv, causal=True)
    except Exception as ex:  # noqa: BLE001
        out["flash_attn_2"] = {"unavailable": str(ex)[:160]}
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from torch.nn.attention.bias import causal_lower_right

    qh = q.transpose(0, 1)[None]                      # [1, Hq, nq, D]
    kh = K.transpose(0, 1)[None].repeat_interleave(HQ // HKV, 1)
    vh = V.transpose(0, 1)[None].repeat_interleave(HQ // HKV, 1)
    bias = causal_lower_right(nq, ctx)
    for name, be in (("sdpa_cudnn", SDPBackend.CUDNN_ATTENTION), ("sdpa_flash", SDPBackend.FLASH_ATTENTION)):
        def f(be=be):
            with sdpa_kernel(be):
                return torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, attn_mask=bias)
        fns[name] = f
    try:
        import flashinfer

        fns["flashinfer"] = lambda: flashinfer.single_prefill_with_kv_cache(q, K, V, causal=True)
    except Exception as ex:  # noqa: BLE001
        out["flashinfer"] = {"unavailable": str(ex)[:160]}
    ref = None
    for name, fn in fns.items():
        try:
            t = dev_time(fn)
            r = fn()
            torch.cuda.synchronize()
            if name == "ours_paged":
                ref = o.float().clone()
                err = 0.0
            else:
                rr = r if not isinstance(r, tuple) else r[0]
                rr = rr[0].transpose(0, 1) if rr.dim() == 4 and rr.shape[1] == HQ else rr.reshape(nq, HQ, HD)
                err = (rr.float() - ref).abs().max().item() if ref is not None else None
            out[name] = {"us": round(1e6 * t, 1), "tflops": round(flops / t / 1e12, 1),
                         "frac_bf16_peak": round(flops / t / 1e12 / PEAK, 4), "max_abs_vs_ours": err}
        except Exception as ex:  # noqa: BLE001
            out[name] = {"error": str(ex)[:200]}
    res[key] = out
    del c, rows, q, o, K, V, qh, kh, vh
    torch.cuda.empty_cache()
res["peak_tflops"] = PEAK
print(json.dumps(res, indent=1))
