#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 python -u -m pytest tests/test_prefill_attention_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 200 python -u profiles/drivers/prefill.py 2>&1 | tail
