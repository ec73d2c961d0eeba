#!/bin/bash
# Compile-time variants of the 128-key prefill kernel.
cd "$(dirname "$0")/.."
for v in "$@"; do
  rm -f paper_2412_12488_b200/_lib/obj/prefill_attn.cu.o
  MKV_NVCC_EXTRA="$v" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null 2>&1
  echo "variant [$v]"
  timeout 120 python -m pytest tests/test_prefill_attention_gpu.py -x -q -p no:cacheprovider -k "not variants" 2>&1 | tail -1
  CASES=8192:6554,8192:0,32768:26214 REPS=10 timeout 120 python profiles/drivers/prefill.py 2>&1 | cut -c1-90
done
rm -f paper_2412_12488_b200/_lib/obj/prefill_attn.cu.o
python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
