#!/bin/bash
# Compile-time A/B of the page-chunk decode kernel: tests + timings per variant.
cd "$(dirname "$0")/.."
for v in "$@"; do
  rm -f paper_2412_12488_b200/_lib/obj/decode_pages.cu.o
  MKV_NVCC_EXTRA="$v" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null 2>&1
  echo "variant [$v]"
  timeout 300 python -m pytest tests/test_decode_attention_gpu.py tests/test_attention_bench_shapes_gpu.py -x -q -p no:cacheprovider -k decode 2>&1 | tail -1
  CASES=${CASES:-1x4096,1x8192,1x32768,4x8192,8x8192,32x8192,8x32768} timeout 300 python profiles/drivers/decode.py
done
rm -f paper_2412_12488_b200/_lib/obj/decode_pages.cu.o
python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
