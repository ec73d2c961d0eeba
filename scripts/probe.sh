#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -u -m pytest tests/test_decode_attention_gpu.py -q -p no:cacheprovider 2>&1 | tail -2
CASES=1x8192,8x8192,32x8192,128x4096,8x32768,1x32768,4x8192 timeout 300 python -u profiles/drivers/decode.py 2>&1 | tail -7
for c in 1x8192 8x8192; do
CASES=$c REPS=5 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_decode_combine python -u profiles/drivers/decode.py 2>&1 | grep -E "gpu__time" | tail -1
done
