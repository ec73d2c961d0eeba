#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f paper_2412_12488_b200/_lib/obj/prefill_attn.cu.o
MKV_NVCC_EXTRA="-DPF_TRACE" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
CASES=8192:6554 REPS=1 timeout 120 python profiles/drivers/prefill.py 2>&1 | tail -2
wc -l gpurun_out/pf_trace.txt
rm -f paper_2412_12488_b200/_lib/obj/prefill_attn.cu.o
