"""Profiling driver: device CRC-32 and KV write frames at the Llama-3.1-70B
KV shape (W = 512 words = 4 KiB per token-layer row).  CUDA-event device
times over back-to-back launches gated behind a sleep kernel.

  crc32      k_crc32 over n bytes of HBM (algorithmic bytes = n read)
  frame_dev  ss_encode_write_frame_async: gather (k_copy_rows) + k_crc32
             into a device frame (algorithmic bytes = 2 n + n: gather read
             + write, CRC read)
  frame_host ss_encode_write_frame into host memory (+ D2H over PCIe)
  receive    ss_receive_write_frame of a host frame (H2D + CRC + apply)
TOKENS=..., REPS=..."""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_12488_b200 import BatchEntry, KVCache  # noqa: E402

W = 512
reps = int(os.environ.get("REPS", "20"))


def timed(fn, s, n_reps=reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        torch.cuda._sleep(50_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n_reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / n_reps


def main():
    s = torch.cuda.Stream()
    E = KVCache(num_pages=8, page_size=16, layers=1, dim=8, device=0)
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    for n in (1 << 16, 1 << 20, 33_550_336, 268_435_456, 2_684_026_880):
        buf = torch.empty(n, dtype=torch.uint8, device="cuda").random_(0, 256)
        t = timed(lambda: E.crc32_async(buf.data_ptr(), n, out.data_ptr(), s.cuda_stream), s)
        print(f"crc32 n={n:>11d}  {t*1e6:9.1f} us  {n/t/1e9:8.1f} GB/s read", flush=True)
        del buf
        torch.cuda.empty_cache()
    for tokens in [int(x) for x in os.environ.get("TOKENS", "1024,8191").split(",")]:
        pages = tokens // 16 + 8
        P = KVCache(num_pages=pages, page_size=16, layers=1, dim=W, device=0, rank=0)
        D = KVCache(num_pages=pages, page_size=16, layers=1, dim=W, device=0, rank=1)
        prompt = np.random.default_rng(1).integers(0, 256, tokens + 1).astype(np.int32)
        P.CreateSequence(1, prompt)
        P.EnsureAllocated(1, tokens)
        plan = P.BeginForward([BatchEntry(1, (0, tokens))])
        rows = torch.empty(tokens * W, dtype=torch.int64, device="cuda").random_()
        P.append_rows_async(plan, 0, rows.data_ptr(), 0)
        torch.cuda.synchronize()
        plan.close()
        r = D.PrepRecv(1, prompt, -1)
        assert r.addr.token_count == tokens
        payload = tokens * W * 8
        from paper_2412_12488_b200.kvcache import frame_write_header_size
        hdr = frame_write_header_size(len(r.addr.ranges))
        fb = torch.empty(payload + hdr + 64, dtype=torch.uint8, device="cuda")
        off = (-(fb.data_ptr() + hdr)) % 32
        cap = payload + hdr + 64 - off
        t = timed(lambda: P.encode_write_frame_async(1, (0, tokens), 0, 7, r.addr,
                                                     fb.data_ptr() + off, cap, s.cuda_stream), s)
        print(f"frame_dev tokens={tokens:6d} payload={payload/1e6:7.1f} MB  {t*1e6:9.1f} us  "
              f"{payload/t/1e9:8.1f} GB/s payload  {3*payload/t/1e9:8.1f} GB/s HBM", flush=True)
        flen = hdr + payload + 4
        hb = torch.empty(flen, dtype=torch.uint8, pin_memory=True)
        walls = []
        for _ in range(6):
            w0 = time.perf_counter()
            P.encode_write_frame_into(1, (0, tokens), 0, 7, r.addr, hb.data_ptr(), flen)
            walls.append(time.perf_counter() - w0)
        tw = float(np.median(walls[1:]))
        print(f"frame_host(pinned) tokens={tokens:6d}  {tw*1e6:9.1f} us  {payload/tw/1e9:8.1f} GB/s payload",
              flush=True)
        walls = []
        for i in range(5):
            w0 = time.perf_counter()
            ack, st = D.receive_write_frame_from(hb.data_ptr(), flen)
            walls.append(time.perf_counter() - w0)
            assert st == (0 if i == 0 else 1), st
        tw = float(np.median(walls[1:]))
        print(f"receive(pinned) tokens={tokens:6d}  {tw*1e6:9.1f} us  {payload/tw/1e9:8.1f} GB/s payload",
              flush=True)
        del P, D, rows, fb
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
