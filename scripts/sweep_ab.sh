#!/bin/bash
# Compile-time variants of the row-copy kernels on the transfer sweep (small and mid sizes).
cd "$(dirname "$0")/.."
for v in "$@"; do
  rm -f paper_2412_12488_b200/_lib/obj/kernels.cu.o
  MKV_NVCC_EXTRA="$v" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null 2>&1
  echo "variant [$v]"
  SWEEP_N=${SWEEP_N:-16,64,256,1024,4096} timeout 300 python profiles/drivers/sweep.py 2>&1 | cut -c1-110
done
rm -f paper_2412_12488_b200/_lib/obj/kernels.cu.o
python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
