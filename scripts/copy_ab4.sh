#!/bin/bash
# Compile-time variants of the row-copy kernels on DirectSends timed behind a
# sleep gate (profiles/drivers/copy_gate.py; SHAPES="tokens:layers ...",
# default 8192:80), and optionally other drivers (EXTRA_DRIVERS="a.py b.py").
cd "$(dirname "$0")/.."
for v in "$@"; do
  rm -f paper_2412_12488_b200/_lib/obj/kernels.cu.o
  MKV_NVCC_EXTRA="$v" python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null 2>&1
  echo "variant [$v]"
  for shp in ${SHAPES:-8192:80}; do
    timeout 300 python profiles/drivers/copy_gate.py "${shp%:*}" "${shp#*:}" 2>&1 | grep gated
  done
  for d in $EXTRA_DRIVERS; do
    timeout 300 python "profiles/drivers/$d" 2>&1 | tail -3 | cut -c1-600
  done
done
rm -f paper_2412_12488_b200/_lib/obj/kernels.cu.o
python -c "from paper_2412_12488_b200 import build as b; b.build()" > /dev/null
