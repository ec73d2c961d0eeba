#!/bin/bash
# Event timeline of CTA (0, 0) of the prefill kernel (-DPF_TRACE):
# gpurun_out/pf_trace_<variant>.txt, "clock event-code" per line.
cd "$(dirname "$0")/.."
CASE=${CASE:-8192:0}
for v in "$@"; do
  rm -f paper_2412_12488_b200/_lib/obj/prefill_attn.cu.o
  MKV_NVCC_EXTRA="-DPF_TRACE $v" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null 2>&1
  CASES=$CASE REPS=1 timeout 120 python profiles/drivers/prefill.py > /dev/null 2>&1
  tag=$(echo "$v" | tr -c 'A-Za-z0-9=' '_')
  mv gpurun_out/pf_trace.txt "gpurun_out/pf_trace_${tag}.txt"
  echo "variant [$v] $(wc -l < gpurun_out/pf_trace_${tag}.txt) events"
done
rm -f paper_2412_12488_b200/_lib/obj/prefill_attn.cu.o
python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
