#!/bin/bash
# A/B of the prefill kernel layouts (MICROKV_PREFILL_VARIANT, see prefill_attn.cu).
cd "$(dirname "$0")/.."
for v in ${VARIANTS:-128 128p 128s 64 2sm}; do
  echo "MICROKV_PREFILL_VARIANT=$v"
  MICROKV_PREFILL_VARIANT=$v timeout 120 python -m pytest tests/test_prefill_attention_gpu.py -x -q -p no:cacheprovider -k "not variants" 2>&1 | tail -1
  MICROKV_PREFILL_VARIANT=$v timeout 120 python profiles/drivers/prefill.py 2>&1 | cut -c1-100
done
