import torch
for nbytes in (33_554_432, 268_435_456, 536_870_912, 1_073_741_824, 4_294_967_296):
    x = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda").uniform_()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): x.sum()
        torch.cuda.synchronize()
        torch.cuda._sleep(20_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20): x.sum()
        e1.record(s)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / 20
    print(f"read {nbytes/1e6:8.1f} MB  {t*1e6:8.1f} us  {nbytes/t/1e9:7.1f} GB/s")
    del x
