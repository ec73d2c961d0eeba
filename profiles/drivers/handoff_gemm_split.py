"""Profiling driver: where does a side-stream send's prefill slowdown come
from at the 8B shape?  bench.py's handoff loop (per layer: one bf16 GEMM of
an 8B layer's FLOPs, the layer's K||V append, the layer's DirectSend behind
its event on a second stream), with every GEMM bracketed by its own events
and the SM clock sampled (NVML) separately for each arm's runs.

Per arm: median GEMM time of layers >= 1 (those overlap the previous layer's
send), median SM clock during the arm, and whole-prefill time; arms rotate
per rep like bench.py.  Usage: handoff_gemm_split.py [8b|70b] [reps]
Env MICROKV_HANDOFF_SEND_PRIO as in bench.py (the arms below also set it
per arm)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2412_12488_b200 import BatchEntry, KVCache  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "8b"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 21
if shape == "8b":
    layers, n_prompt, k, n = 32, 4096, 4096, 53248
else:
    layers, n_prompt, k, n = bench.L, bench.PROMPT, 8192, 104448
W, PAGE = bench.W, bench.PAGE
e = n_prompt - 1
prompt = [int(x) for x in np.random.Generator(np.random.MT19937(4)).integers(0, 256, n_prompt)]
pages = n_prompt // PAGE + 16
P = KVCache(num_pages=pages, page_size=PAGE, layers=layers, dim=W, device=0, rank=0)
D = KVCache(num_pages=pages, page_size=PAGE, layers=layers, dim=W, device=0, rank=1)
P.attach_peer(1, D)
X = torch.randn(e, k, device="cuda", dtype=torch.bfloat16)
Wt = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) * 0.01
Y = torch.empty(e, n, device="cuda", dtype=torch.bfloat16)
rows = torch.randint(-2**62, 2**62, (e * W,), dtype=torch.int64, device="cuda")
cs = torch.cuda.Stream()
streams = {-1: torch.cuda.Stream(priority=-1), 0: torch.cuda.Stream(priority=0)}
ds = torch.cuda.Stream()
# (name, mover mode or None, ctas, send stream priority)
ARMS = [("none", None, 0, 0), ("kernel_full", 0, 0, -1), ("kernel_32ctas", 0, 32, -1),
        ("kernel_32ctas_prio0", 0, 32, 0), ("kernel_full_prio0", 0, 0, 0),
        ("write_through", "fused", 0, 0)]
res = {a[0]: {"prefill_ms": [], "gemm_us": [], "clock_mhz": [], "reasons": set(), "mcycles": []}
       for a in ARMS}
seq = 10
for rep in range(reps + 1):
    order = ARMS[rep % len(ARMS):] + ARMS[:rep % len(ARMS)]
    for name, mode, ctas, prio in order:
        send, fused = mode is not None, mode == "fused"
        ms = streams[prio]
        seq += 1
        if send:
            P.set_send_mode(0 if fused else mode, ctas)
            r = D.PrepRecv(seq, prompt, -1)
        P.CreateSequence(seq, prompt)
        P.EnsureAllocated(seq, e)
        plan = P.BeginForward([BatchEntry(seq, (0, e))])
        dplan = P.begin_direct_send(seq, (0, e), 1, r.addr, 7) if send else None
        torch.cuda.synchronize()
        g0 = [torch.cuda.Event(enable_timing=True) for _ in range(layers)]
        g1 = [torch.cuda.Event(enable_timing=True) for _ in range(layers)]
        done = [torch.cuda.Event() for _ in range(layers)]
        sampler = bench.ClockSampler(0)
        sampler.__enter__()
        for layer in range(layers):
            g0[layer].record(cs)
            with torch.cuda.stream(cs):
                torch.matmul(X, Wt, out=Y)
            g1[layer].record(cs)
            if fused:
                P.append_rows_send_async(plan, dplan, (layer, layer + 1), rows.data_ptr(),
                                         cs.cuda_stream)
            else:
                P.append_rows_async(plan, layer, rows.data_ptr(), cs.cuda_stream)
                done[layer].record(cs)
                if send:
                    P.launch_direct_send_after_async(dplan, (layer, layer + 1),
                                                     done[layer].cuda_event, ms.cuda_stream)
        torch.cuda.synchronize()
        sampler.__exit__(None, None, None)
        P.synchronize()
        if rep > 0:
            rr = res[name]
            t_ms = g0[0].elapsed_time(g1[-1])
            rr["prefill_ms"].append(t_ms)
            if sampler.samples:  # clock-normalised: ms x mean MHz = Mcycles at the sampled clock
                rr["mcycles"].append(t_ms * float(np.mean(sampler.samples)) / 1e3)
            rr["gemm_us"] += [1e3 * g0[i].elapsed_time(g1[i]) for i in range(1, layers)]
            rr["clock_mhz"] += sampler.samples
            rr["reasons"] |= sampler.reasons
        if send:
            D.wait_receive_async(seq, 60000, ds.cuda_stream)
            ds.synchronize()
            D.synchronize()
            assert D.DrainReceiveCompletions() == [seq]
            D.FreeSequence(seq)
            dplan.close()
        plan.close()
        P.FreeSequence(seq)
P.set_send_mode(0, 0)
base = float(np.median(res["none"]["prefill_ms"]))
cbase = float(np.median(res["none"]["mcycles"])) if res["none"]["mcycles"] else None
gbase = float(np.median(res["none"]["gemm_us"]))
out = {"shape": shape, "layers": layers, "reps": reps, "gemm": f"X[{e},{k}] @ W[{k},{n}]"}
for name, rr in res.items():
    g = np.array(rr["gemm_us"])
    c = np.array(rr["clock_mhz"]) if rr["clock_mhz"] else np.array([0])
    out[name] = {"prefill_ms_median": round(float(np.median(rr["prefill_ms"])), 3),
                 "slowdown_pct": round(100 * (float(np.median(rr["prefill_ms"])) / base - 1), 2),
                 "slowdown_pct_clock_normalised": (
                     round(100 * (float(np.median(rr["mcycles"])) / cbase - 1), 2)
                     if cbase and rr["mcycles"] else None),
                 "slowdown_pct_paired": round(float(np.median(
                     [100 * (x / y - 1) for x, y in zip(rr["prefill_ms"], res["none"]["prefill_ms"])])), 2),
                 "gemm_us_median": round(float(np.median(g)), 1),
                 "gemm_us_p10_p90": [round(float(np.percentile(g, 10)), 1),
                                     round(float(np.percentile(g, 90)), 1)],
                 "gemm_slowdown_pct": round(100 * (float(np.median(g)) / gbase - 1), 2),
                 "sm_mhz_median": float(np.median(c)),
                 "sm_mhz_p10": float(np.percentile(c, 10)),
                 "clock_samples": int(len(rr["clock_mhz"])),
                 "reasons": sorted(rr["reasons"])}
print(json.dumps(out, indent=1))
