#!/bin/bash
cd "$(dirname "$0")/.."
python - <<'PY'
import sys, json, torch
sys.path.insert(0, '.')
import bench
print(json.dumps(bench.measure_engine(torch)))
PY
