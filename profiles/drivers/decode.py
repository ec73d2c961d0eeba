"""Profiling driver: paged GQA decode attention (70B: Hq=64, Hkv=8, D=128)
over a sweep of (batch, ctx); device time gated behind a sleep kernel so the
launches run back to back.  MICROKV_DECODE_GRID caps the stream-K grid (tuning)."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import json  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_12488_b200.kvcache as kc  # noqa: E402

if "--lib" in sys.argv:  # A/B of a variant build
    kc.PRODUCT_LIB = Path(sys.argv[sys.argv.index("--lib") + 1]).resolve()
from paper_2412_12488_b200 import BatchEntry, KVCache  # noqa: E402

HQ, HKV, HD, W = 64, 8, 128, 512
try:
    peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
except Exception:
    peak = 6650.0
cases = [(int(b), int(c)) for b, c in (x.split("x") for x in
         os.environ.get("CASES", "1x8192,8x8192,32x8192,128x4096,8x32768").split(","))]
for B, ctx in cases:
    # Launches cycle over enough layers to exceed L2 (126 MB): HBM reads.
    L = max(1, min(16, -(-300_000_000 // (B * ctx * 4096))))
    c = KVCache(num_pages=B * (ctx // 16) + 16, page_size=16, layers=L, dim=W, device=0)
    for b in range(B):
        c.CreateSequence(b, np.zeros(ctx, np.int32))
        c.EnsureAllocated(b, ctx)
    plan = c.BeginForward([BatchEntry(b, (0, ctx)) for b in range(B)])
    rows = (torch.randn(B * ctx * W * 4, device="cuda") * 0.5).to(torch.bfloat16)
    for layer in range(L):
        c.append_rows_async(plan, layer, rows.data_ptr(), 0)
    torch.cuda.synchronize()
    plan.close()
    del rows
    d = c.begin_decode(list(range(B)), [ctx] * B)
    q = torch.randn(B, HQ, HD, device="cuda", dtype=torch.bfloat16)
    o = torch.empty_like(q)
    s = torch.cuda.Stream()
    for _ in range(3):
        c.paged_decode_attention_async(d, 0, HQ, HKV, HD, HD ** -0.5, q.data_ptr(), o.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    reps = int(os.environ.get("REPS", "20"))
    with torch.cuda.stream(s):
        torch.cuda._sleep(20_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(reps):
        c.paged_decode_attention_async(d, i % L, HQ, HKV, HD, HD ** -0.5, q.data_ptr(), o.data_ptr(), s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    alg = B * ctx * 4096 + 2 * q.numel() * 2
    print(f"B={B:4d} ctx={ctx:6d}  {t*1e6:8.1f} us  {alg/t/1e9:7.1f} GB/s  {alg/t/1e9/peak:.3f} of peak")
    d.close()
    del c
    torch.cuda.empty_cache()
