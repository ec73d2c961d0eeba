#!/bin/bash
# A/B of the prefill kernels: the single-CTA kernel and the 2-SM pair kernel.
cd "$(dirname "$0")/.."
for v in 1 0; do
  echo "MICROKV_PREFILL_2SM=$v"
  MICROKV_PREFILL_2SM=$v timeout 120 python -m pytest tests/test_prefill_attention_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
  MICROKV_PREFILL_2SM=$v timeout 120 python profiles/drivers/prefill.py 2>&1 | cut -c1-100
done
