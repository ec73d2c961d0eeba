"""Profiling driver: bench.py's config-4 prefix migration alone (fan-out,
sequential DirectSends, relay chain; 70B shape, 8K prefix, 3 targets)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402

print(json.dumps(bench.measure_prefix_migration(torch), indent=1))
