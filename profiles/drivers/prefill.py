"""Profiling driver: tcgen05 paged causal prefill attention (70B: Hq=64,
Hkv=8, D=128) over (ctx, q_begin) cases; device time with CUDA events over
back-to-back launches gated behind a sleep kernel.  Causal FLOPs =
4 * D * Hq * sum_{p=q_begin}^{ctx-1} (p + 1).  For scale, the same attention
through torch SDPA (library flash/cuDNN kernels) on contiguous, already
gathered K/V is timed beside it when available (no paging, not the product).
CASES="ctx:q_begin,..."; REPS; HQ / HKV (default 64 / 8, Llama 70B; 32 / 8 for 8B)."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_12488_b200 import BatchEntry, KVCache  # noqa: E402

HQ, HKV, HD = int(os.environ.get("HQ", "64")), int(os.environ.get("HKV", "8")), 128
W = 4 * HKV * HD // 8
try:  # driver-measured burst bf16 peak (MEASURED_PEAKS.json), as bench.py uses
    import json as _json
    PEAK = float(_json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops"])
except Exception:
    PEAK = 1624.4
cases = [(int(a), int(b)) for a, b in (x.split(":") for x in
         os.environ.get("CASES", "8192:6554,8192:0,4096:0,32768:26214,2048:0").split(","))]
reps = int(os.environ.get("REPS", "10"))


def timed(fn, s):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        torch.cuda._sleep(20_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


for ctx, qb in cases:
    nq = ctx - qb
    c = KVCache(num_pages=ctx // 16 + 16, page_size=16, layers=1, dim=W, device=0)
    c.CreateSequence(1, np.zeros(ctx, np.int32))
    c.EnsureAllocated(1, ctx)
    plan = c.BeginForward([BatchEntry(1, (0, ctx))])
    rows = (torch.randn(ctx, 2, HKV, HD, device="cuda") * 0.5).to(torch.bfloat16)
    c.append_rows_async(plan, 0, rows.data_ptr(), 0)
    torch.cuda.synchronize()
    plan.close()
    q = (torch.randn(nq, HQ, HD, device="cuda") * 0.5).to(torch.bfloat16)
    o = torch.empty_like(q)
    s = torch.cuda.Stream()
    flops = 4.0 * HD * HQ * (sum(range(qb + 1, ctx + 1)))
    t = timed(lambda: c.paged_prefill_attention_async(1, (qb, ctx), 0, HQ, HKV, HD, HD ** -0.5,
                                                      q.data_ptr(), o.data_ptr(), s.cuda_stream), s)
    line = (f"ctx={ctx:6d} q=[{qb},{ctx}) nq={nq:6d}  {t*1e6:9.1f} us  {flops/t/1e12:7.1f} TFLOP/s "
            f" {flops/t/1e12/PEAK:.3f} of bf16 peak")
    try:
        from torch.nn.attention.bias import causal_lower_right
        qs = q.transpose(0, 1).unsqueeze(0)                       # [1, Hq, nq, D]
        ks = rows[:, 0].transpose(0, 1).unsqueeze(0).repeat_interleave(HQ // HKV, 1).contiguous()
        vs = rows[:, 1].transpose(0, 1).unsqueeze(0).repeat_interleave(HQ // HKV, 1).contiguous()
        mask = causal_lower_right(nq, ctx)
        with torch.cuda.stream(s):
            ts = timed(lambda: torch.nn.functional.scaled_dot_product_attention(
                qs, ks, vs, attn_mask=mask), s)
        line += f" | torch SDPA (contiguous) {ts*1e6:9.1f} us {flops/ts/1e12:7.1f} TFLOP/s"
    except Exception as e:  # noqa: BLE001
        line += f" | SDPA n/a ({type(e).__name__})"
    print(line, flush=True)
    del c
    torch.cuda.empty_cache()
