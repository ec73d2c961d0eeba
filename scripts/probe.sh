#!/bin/bash
# tcgen05 prefill probe + prefill attention tests, each bounded; unbuffered.
cd "$(dirname "$0")/.."
timeout 60 ./profiles/micro/tc_probe 4 40 0; echo "rc=$?"
timeout 60 ./profiles/micro/tc_probe 4 300 0; echo "rc=$?"
timeout 60 ./profiles/micro/tc_probe 4 1000 800; echo "rc=$?"
timeout 300 python -u -m pytest tests/test_prefill_attention_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -20
timeout 200 python -u profiles/drivers/prefill.py 2>&1 | tail
