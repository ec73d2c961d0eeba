"""Profiling driver: the per-layer KV append with and without the layer's
remote_send, at the 70B and 8B KV shapes (P and D on one GPU).

Modes, each over every layer of one request, launches back to back on one
stream behind a sleep kernel (device time per layer from CUDA events around
each call, median over layers and reps):
  append          ss_append_rows_async alone (the no-send baseline)
  append+send     ss_append_rows_async then ss_launch_direct_send_async
  fused           ss_append_rows_send_async (write-through)
Bytes: append = 2 x rows x 4 KiB (read + write); the send adds a read and a
write of the same rows; fused reads once and writes twice (3 x).
Usage: append_send.py [70b|8b|both] [reps]"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2412_12488_b200 import BatchEntry, KVCache  # noqa: E402

W, PAGE = 512, 16


def peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6650.0


def run(L, n_prompt, reps):
    e = n_prompt - 1
    pages = n_prompt // PAGE + 16
    P = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=0)
    D = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    rng = np.random.default_rng(3)
    prompt = [int(x) for x in rng.integers(0, 256, n_prompt)]
    rows = [torch.randint(-2**62, 2**62, (e, W), dtype=torch.int64, device="cuda") for _ in range(L)]
    s = torch.cuda.Stream()
    out = {}
    seq = 100
    for mode in ("append", "append+send", "fused"):
        per_layer = []
        for rep in range(reps + 1):
            seq += 1
            P.CreateSequence(seq, prompt)
            P.EnsureAllocated(seq, e)
            fplan = P.BeginForward([BatchEntry(seq, (0, e))])
            send = mode != "append"
            if send:
                r = D.PrepRecv(seq, prompt, -1)
                dplan = P.begin_direct_send(seq, (0, e), 1, r.addr, rep)
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(L + 1)]
            with torch.cuda.stream(s):
                torch.cuda._sleep(2_000_000)
            for layer in range(L):
                ev[layer].record(s)
                if mode == "fused":
                    P.append_rows_send_async(fplan, dplan, (layer, layer + 1), rows[layer].data_ptr(),
                                             s.cuda_stream)
                else:
                    P.append_rows_async(fplan, layer, rows[layer].data_ptr(), s.cuda_stream)
                    if send:
                        P.launch_direct_send_async(dplan, (layer, layer + 1), s.cuda_stream)
            ev[L].record(s)
            s.synchronize()
            P.synchronize()
            if rep > 0:
                per_layer += [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(L)]
            if send:
                assert D.DrainReceiveCompletions() == [seq]
                D.FreeSequence(seq)
                dplan.close()
            fplan.close()
            P.FreeSequence(seq)
        us = float(np.median(per_layer))
        traffic = (2 if mode == "append" else (4 if mode == "append+send" else 3)) * e * W * 8
        out[mode] = {"us_per_layer": round(us, 2), "p10_us": round(float(np.percentile(per_layer, 10)), 2),
                     "p90_us": round(float(np.percentile(per_layer, 90)), 2),
                     "gbs": round(traffic / us / 1e3, 1), "hbm_frac": round(traffic / us / 1e3 / peak(), 4)}
    out["fused_extra_us"] = round(out["fused"]["us_per_layer"] - out["append"]["us_per_layer"], 2)
    del P, D, rows
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "both"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    res = {}
    if which in ("70b", "both"):
        res["70b"] = run(80, 8192, reps)
    if which in ("8b", "both"):
        res["8b"] = run(32, 4096, reps)
    print(json.dumps(res, indent=1))
