"""Profiling driver: the router strategies over B200 engines (bench.measure_router)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402

print(json.dumps(bench.measure_router(torch), indent=1))
