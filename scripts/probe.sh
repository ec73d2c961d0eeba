#!/bin/bash
cd "$(dirname "$0")/.."
python - <<'PY'
import sys, json, torch
sys.path.insert(0, '.')
import bench
for i in range(3):
    for after in (True, False):
        r = bench.measure_handoff_gemm(torch, 32, 4096, 4096, 53248, "8B", after)
        print("8B after" if after else "8B plain", r["exposed_tail_us"], r["slowdown_pct"], r["prefill_ms_without_sends"])
for after in (True, False):
    r = bench.measure_handoff_gemm(torch, after=after)
    print("70B after" if after else "70B plain", r["exposed_tail_us"], r["slowdown_pct"])
PY
