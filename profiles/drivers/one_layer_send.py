"""Profiling driver: one-layer DirectSends at the 70B shape (for launch lists)."""
import sys
sys.path.insert(0, '.')
import torch, bench
import numpy as np
from paper_2412_12488_b200 import KVCache
L, W, PAGE, PROMPT = bench.L, bench.W, bench.PAGE, bench.PROMPT
prompt = bench._prompt(8)
e = PROMPT - 1
pages = PROMPT // PAGE + 16
P = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=0)
D = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=1)
P.attach_peer(1, D)
bench._populate_prefix_l(P, 1, prompt, torch, L)
s = torch.cuda.Stream()
for rep in range(6):
    r = D.PrepRecv(600 + rep, prompt, -1)
    plan = P.begin_direct_send(1, (0, e), 1, r.addr, rep)
    with torch.cuda.stream(s):
        torch.cuda._sleep(4_000_000)
    P.launch_direct_send_async(plan, (0, 1), s.cuda_stream)
    s.synchronize()
    plan.close()
    D.FreeSequence(600 + rep)
print("done")
