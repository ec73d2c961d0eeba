#!/bin/bash
# A/B of k_copy_rows compile-time variants: the 80-layer DirectSend
# (copy_time.py) and the per-layer append / gather (append_gather.py).
cd "$(dirname "$0")/.."
for v in "$@"; do
  rm -f paper_2412_12488_b200/_lib/obj/kernels.cu.o
  MKV_NVCC_EXTRA="$v" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null 2>&1
  for rep in 1 2; do
    echo "variant [$v] directsend: $(timeout 300 python profiles/drivers/copy_time.py 2>&1 | tail -1)"
    echo "variant [$v] append/gather: $(timeout 300 python profiles/drivers/append_gather.py 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
rm -f paper_2412_12488_b200/_lib/obj/kernels.cu.o
python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
