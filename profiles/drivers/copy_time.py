"""Profiling driver: device time of DirectSend launches (80 layers x 8191
rows, 70B shape, P and D on one GPU), CUDA events around back-to-back
launches into fresh receive windows; no completion checks (usable with
measurement-only builds such as -DMKV_NO_FILL)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_12488_b200 import KVCache  # noqa: E402

L, W, P, n = 80, 512, 16, 8192
rng = np.random.Generator(np.random.MT19937(1))
prompt = [int(x) for x in rng.integers(0, 256, n)]
Pe = KVCache(num_pages=n // P + 16, page_size=P, layers=L, dim=W, device=0, rank=0)
D = KVCache(num_pages=4 * (n // P) + 16, page_size=P, layers=L, dim=W, device=0, rank=1)
Pe.attach_peer(1, D)
r = Pe.PrepRecv(1, prompt, n)
buf = torch.randint(-2**62, 2**62, (n * W,), dtype=torch.int64, device="cuda")
for layer in range(L):
    Pe.apply_remote_write_async(r.addr, layer, buf.data_ptr(), n * W, 0, 0)
torch.cuda.synchronize()
Pe.synchronize()
Pe.DrainReceiveCompletions()
s = torch.cuda.Stream()
times = []
for i in range(8):
    rr = D.PrepRecv(100 + i, prompt, -1)
    plan = Pe.begin_direct_send(1, (0, n - 1), 1, rr.addr, i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    Pe.launch_direct_send_async(plan, (0, L), s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1) / 1e3)
    plan.close()
    D.DrainReceiveCompletions()
    D.FreeSequence(100 + i)
t = float(np.median(times[2:]))
payload = (n - 1) * L * W * 8
print(f"DirectSend {t*1e6:.1f} us  {payload/t/1e9:.1f} GB/s payload  {2*payload/t/1e9/6551.7:.3f} of HBM copy peak")
