#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests/test_prefill_attention_gpu.py -q -p no:cacheprovider 2>&1 | tail -2
VARIANTS="128 64" bash scripts/pf_ab.sh
