"""Profiling driver: bench.py's append/gather measurement and the send
movers alone (70B shape, 8192 rows x 80 layers).  `--lib PATH` runs a
variant build of the product library (A/B of compile-time switches)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2412_12488_b200.kvcache as kc  # noqa: E402

if "--lib" in sys.argv:
    kc.PRODUCT_LIB = Path(sys.argv[sys.argv.index("--lib") + 1]).resolve()
import bench  # noqa: E402

bench.SEND_ARMS = bench.SEND_ARMS[:1]
print(json.dumps({"lib": str(kc.PRODUCT_LIB), "append_gather": bench.measure_append_gather(torch),
                  "send": bench.measure_send_modes(torch)}))
