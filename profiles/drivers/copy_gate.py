"""Profiling driver: the headline DirectSend launch (80 layers x 8191 rows,
70B shape, P and D on one GPU) timed two ways with CUDA events: as bench.py
does (the stream idle at the first event, so the window also holds the
host's enqueue of validation + copy) and behind a ~60 us sleep kernel
enqueued first (the window holds device work only).  Prints both and the
difference (host enqueue latency seen by the device)."""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_12488_b200 import KVCache  # noqa: E402

W, P = 512, 16
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192   # prompt tokens (n - 1 sent)
L = int(sys.argv[2]) if len(sys.argv) > 2 else 80     # layers
rng = np.random.Generator(np.random.MT19937(1))
prompt = [int(x) for x in rng.integers(0, 256, n)]
extra = n // P // 2 + 16 if os.environ.get("FRAGMENT") else 16
Pe = KVCache(num_pages=n // P + extra, page_size=P, layers=L, dim=W, device=0, rank=0)
D = KVCache(num_pages=n // P + extra, page_size=P, layers=L, dim=W, device=0, rank=1)
Pe.attach_peer(1, D)
if os.environ.get("FRAGMENT"):  # shuffle both free lists: interleaved 3-page sequences, every other freed
    for c in (Pe, D):
        for i in range(n // P // 3 // 2):
            c.CreateSequence(50000 + i, [1] * (3 * P))
            c.EnsureAllocated(50000 + i, 3 * P)
        for i in range(0, n // P // 3 // 2, 2):
            c.FreeSequence(50000 + i)
r = Pe.PrepRecv(1, prompt, n)
buf = torch.randint(-2**62, 2**62, (n * W,), dtype=torch.int64, device="cuda")
for layer in range(L):
    Pe.apply_remote_write_async(r.addr, layer, buf.data_ptr(), n * W, 0, 0)
torch.cuda.synchronize()
Pe.synchronize()
Pe.DrainReceiveCompletions()
s = torch.cuda.Stream()
res = {"idle": [], "gated": []}
host_us = []
for i in range(16 if n * L > 300000 else 40):
    mode = "gated" if i % 2 else "idle"
    rr = D.PrepRecv(100 + i, prompt, -1)
    plan = Pe.begin_direct_send(1, (0, n - 1), 1, rr.addr, i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if mode == "gated":
        with torch.cuda.stream(s):
            torch.cuda._sleep(120000)
    e0.record(s)
    h0 = time.perf_counter()
    Pe.launch_direct_send_async(plan, (0, L), s.cuda_stream)
    host_us.append(1e6 * (time.perf_counter() - h0))
    e1.record(s)
    torch.cuda.synchronize()
    if i >= 4:
        res[mode].append(e0.elapsed_time(e1) * 1e3)
    plan.close()
    assert D.DrainReceiveCompletions() == [100 + i]
    D.FreeSequence(100 + i)
payload = (n - 1) * L * W * 8
for k, v in res.items():
    t = float(np.median(v))
    print(f"n={n} L={L} {k:6s} {t:8.1f} us  (range {min(v):.1f}-{max(v):.1f})  {2*payload/t/1e3/6551.7:.4f} of the HBM copy peak")
print(f"host enqueue of launch_direct_send_async: median {np.median(host_us[4:]):.1f} us")
