#!/bin/bash
cd "$(dirname "$0")/.."
python -u profiles/drivers/readbw.py
CASES=1x8192,4x8192,8x8192,16x8192,1x32768,32x8192,128x4096,8x32768 timeout 300 python -u profiles/drivers/decode.py 2>&1 | tail -8
