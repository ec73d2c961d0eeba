#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
python - <<'PY'
import sys, json, torch
sys.path.insert(0, '.')
import bench
print(json.dumps(bench.measure_handoff_gemm(torch)))
print(json.dumps(bench.measure_handoff_gemm(torch, 32, 4096, 4096, 53248, "8B")))
PY
