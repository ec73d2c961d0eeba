"""Profiling driver: plain read bandwidth (torch.sum over fp32) by size, the
launches cycling over enough buffers to exceed L2 (126 MB), CUDA events
over back-to-back launches behind a sleep kernel."""
import torch

for nbytes in (33_554_432, 268_435_456, 536_870_912, 1_073_741_824, 4_294_967_296):
    nbuf = max(1, min(16, -(-300_000_000 // nbytes)))
    xs = [torch.empty(nbytes // 4, dtype=torch.float32, device="cuda").uniform_() for _ in range(nbuf)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for x in xs: x.sum()
        torch.cuda.synchronize()
        torch.cuda._sleep(20_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(20): xs[i % nbuf].sum()
        e1.record(s)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / 20
    print(f"read {nbytes/1e6:8.1f} MB  {t*1e6:8.1f} us  {nbytes/t/1e9:7.1f} GB/s")
    del xs
