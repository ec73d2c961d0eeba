"""Profiling driver: bench.py's handoff measurement alone (70B or 8B shape),
the no-send arm and the send arms of SEND_ARMS, per-rep numbers; SM clock
samples beside it.  Usage: handoff.py [8b|8b-one-rotation|70b|70b-split] [reps] [arm,arm,...]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "8b"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 9
if len(sys.argv) > 3:
    keep = sys.argv[3].split(",")
    bench.SEND_ARMS = tuple(a for a in bench.SEND_ARMS if a[0] in keep)
sampler = bench.ClockSampler(0)
sampler.__enter__()
if shape == "8b":
    r = bench.measure_handoff_8b(torch, reps=reps)
elif shape == "8b-one-rotation":  # every arm in one rotation (the copy-engine arm perturbs it)
    r = bench.measure_handoff_gemm(torch, 32, 4096, 4096, 53248, "8B", reps=reps)
elif shape == "70b-split":  # K||V from the layer's first 20% of FLOPs
    r = bench.measure_handoff_gemm(torch, reps=reps, kv_share=0.2)
else:
    r = bench.measure_handoff_gemm(torch, reps=reps)
sampler.__exit__(None, None, None)
r["clocks"] = sampler.summary()
print(json.dumps(r, indent=1))
