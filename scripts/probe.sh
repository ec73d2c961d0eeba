#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_prefill_attention_gpu.py -q -p no:cacheprovider 2>&1 | tail -3
CASES=2048:1638,4096:3276,8192:6553,16384:13107,8192:0,2048:0 python profiles/drivers/prefill.py 2>&1 | cut -c1-110
for sp in 1 2 3 4; do echo "split $sp"; MICROKV_PREFILL_SPLIT=$sp CASES=2048:1638,4096:3276 python profiles/drivers/prefill.py 2>&1 | cut -c1-80; done
