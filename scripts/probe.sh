#!/bin/bash
cd "$(dirname "$0")/.."
for v in "" "-DMKV_LD_NO_EF"; do
  rm -f paper_2412_12488_b200/_lib/obj/kernels.cu.o
  MKV_NVCC_EXTRA="$v" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null 2>&1
  python - <<PY
import sys, json, torch
sys.path.insert(0, '.')
import bench
print("[$v]", json.dumps(bench.measure_append_gather(torch)))
PY
done
rm -f paper_2412_12488_b200/_lib/obj/kernels.cu.o
python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
