#!/bin/bash
# Per-warp phase sums of the prefill softmax (build with -DPF_PROF): wait for S,
# S load, row max, P half 1 (+rescale, store), P half 2 (+store), clk.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f paper_2412_12488_b200/_lib/obj/prefill_attn.cu.o
MKV_NVCC_EXTRA="-DPF_PROF" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
CASES=${CASES:-8192:6554} REPS=1 timeout 120 python profiles/drivers/prefill.py 2>&1 | tail -1
cat gpurun_out/pf_prof.txt
rm -f paper_2412_12488_b200/_lib/obj/prefill_attn.cu.o
python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
