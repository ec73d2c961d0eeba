"""Profiling driver: the transfer sweep of bench.py (config 5: DirectSend of
n tokens x 80 layers at the 70B shape, P and D on one GPU), device time per
migration and API wall time."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402

for k, v in bench.measure_sweep(torch).items():
    print(k, v, flush=True)
