#!/bin/bash
# Per-warp phase sums of the prefill kernel (-DPF_PROF): cycles waiting for S,
# loading S from TMEM, row max, first / second half of P, for the heaviest
# CTA of each KV head; one line per softmax warp (gpurun_out/pf_prof*.txt).
cd "$(dirname "$0")/.."
CASE=${CASE:-8192:0}
for v in "$@"; do
  rm -f paper_2412_12488_b200/_lib/obj/prefill_attn.cu.o
  MKV_NVCC_EXTRA="-DPF_PROF $v" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null 2>&1
  CASES=$CASE REPS=1 timeout 120 python profiles/drivers/prefill.py > /dev/null 2>&1
  tag=$(echo "$v" | tr -c 'A-Za-z0-9=' '_')
  mv gpurun_out/pf_prof.txt "gpurun_out/pf_prof_${tag}.txt"
  echo "variant [$v]"; head -8 "gpurun_out/pf_prof_${tag}.txt"
done
rm -f paper_2412_12488_b200/_lib/obj/prefill_attn.cu.o
python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
