#!/bin/bash
# A/B of the prefill kernels: variant 1 (default) and the two-tile kernel.
cd "$(dirname "$0")/.."
for v in 0 1; do
  echo "MICROKV_PREFILL_V0=$v"
  MICROKV_PREFILL_V0=$v timeout 200 python -m pytest tests/test_prefill_attention_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
  MICROKV_PREFILL_V0=$v timeout 200 python profiles/drivers/prefill.py 2>&1 | cut -c1-100
done
