#!/bin/bash
# Decode-attention compile-time variants: cp.async ring depth.
cd "$(dirname "$0")/.."
for v in "-DDA_STAGES=2" "-DDA_STAGES=3" "-DDA_STAGES=4"; do
  rm -f paper_2412_12488_b200/_lib/obj/decode_attn.cu.o
  MKV_NVCC_EXTRA="$v" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null 2>&1
  echo "variant [$v]"
  timeout 120 python -m pytest tests/test_decode_attention_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
  CASES=1x8192,8x8192,32x8192,128x4096,8x32768 timeout 120 python profiles/drivers/decode.py
done
rm -f paper_2412_12488_b200/_lib/obj/decode_attn.cu.o
python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
