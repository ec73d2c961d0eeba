"""Profiling driver: one DirectSend plan sent layer by layer (80 launches of
one 70B layer each, back to back behind a sleep) — the per-layer send loop of
a handoff; device time per layer launch."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2412_12488_b200 import KVCache  # noqa: E402

L, W, PAGE, PROMPT = bench.L, bench.W, bench.PAGE, bench.PROMPT
prompt = bench._prompt(8)
e = PROMPT - 1
pages = PROMPT // PAGE + 16
P = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=0)
D = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=1)
P.attach_peer(1, D)
bench._populate_prefix_l(P, 1, prompt, torch, L)
s = torch.cuda.Stream()
ts = []
for rep in range(5):
    r = D.PrepRecv(700 + rep, prompt, -1)
    plan = P.begin_direct_send(1, (0, e), 1, r.addr, rep)
    with torch.cuda.stream(s):
        torch.cuda._sleep(20_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for layer in range(L):
        P.launch_direct_send_async(plan, (layer, layer + 1), s.cuda_stream)
    e1.record(s)
    s.synchronize()
    assert D.DrainReceiveCompletions() == [700 + rep]
    ts.append(e0.elapsed_time(e1) / 1e3 / L)
    plan.close()
    D.FreeSequence(700 + rep)
t = float(np.median(ts[1:]))
print(f"per-layer DirectSend: {t * 1e6:.1f} us per 70B layer ({2 * e * 4096 / t / 1e9:.0f} GB/s read+write)")
