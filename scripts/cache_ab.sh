#!/bin/bash
# Compile-time variants of cache.cc (host-side launch choices) on the sweep and the sends.
cd "$(dirname "$0")/.."
for v in "$@"; do
  rm -f paper_2412_12488_b200/_lib/obj/cache.cc.o
  MKV_CXX_EXTRA="$v" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null 2>&1
  echo "variant [$v]"
  SWEEP_N=${SWEEP_N:-64,256,4096} timeout 300 python profiles/drivers/sweep.py 2>&1 | cut -c1-90
  timeout 300 python profiles/drivers/send_modes.py 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kernel_full', d['kernel_full'])"
done
rm -f paper_2412_12488_b200/_lib/obj/cache.cc.o
python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
