#!/bin/bash
# Register-cap variants of the fan-out (write-through) kernel on the per-layer fused append+send.
cd "$(dirname "$0")/.."
summ() { python -c "
import json,sys
t=sys.stdin.read(); d=json.loads(t[t.index('{'):])
print({k:(v['fused']['us_per_layer'],v['fused']['hbm_frac'],v['append']['us_per_layer']) for k,v in d.items()})"; }
for v in "$@"; do
  rm -f paper_2412_12488_b200/_lib/obj/kernels.cu.o
  MKV_NVCC_EXTRA="$v" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null 2>&1
  echo -n "variant [$v] "
  timeout 300 python profiles/drivers/append_send.py both 3 2>/dev/null | summ
done
rm -f paper_2412_12488_b200/_lib/obj/kernels.cu.o
python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
