"""Profiling driver: the bench's DirectSend migration step (70B KV shape,
8,191 tokens x L layers, P and D on cuda:0), repeated --reps times.

    ncu --set full -k regex:k_copy_rows -s 2 -c 1 -o prof python profiles/drivers/migrate.py
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_12488_b200 import KVCache  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=80)
ap.add_argument("--tokens", type=int, default=8192)
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
L, W, P, n = a.layers, 512, 16, a.tokens
rng = np.random.Generator(np.random.MT19937(1))
prompt = [int(x) for x in rng.integers(0, 256, n)]
Pe = KVCache(num_pages=n // P + 16, page_size=P, layers=L, dim=W, device=0, rank=0)
D = KVCache(num_pages=n // P + 16, page_size=P, layers=L, dim=W, device=0, rank=1)
Pe.attach_peer(1, D)
r = Pe.PrepRecv(1, prompt, n)
buf = torch.randint(-2**62, 2**62, (n * W,), dtype=torch.int64, device="cuda")
for layer in range(L):
    Pe.apply_remote_write_async(r.addr, layer, buf.data_ptr(), n * W, 0, 0)
torch.cuda.synchronize()
Pe.synchronize()
assert Pe.DrainReceiveCompletions() == [1]
s = torch.cuda.Stream()
for i in range(a.reps):
    rr = D.PrepRecv(100 + i, prompt, -1)
    Pe.direct_send_async(1, (0, n - 1), 1, rr.addr, i, (0, L), s.cuda_stream)
    s.synchronize()
    assert D.DrainReceiveCompletions() == [100 + i]
    D.FreeSequence(100 + i)
print("migrate driver done")
