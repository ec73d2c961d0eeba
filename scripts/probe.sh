#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy_rows -s 81 -c 1 \
  -o gpurun_out/prof_copy_rows -f python profiles/drivers/migrate.py --reps 3 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out/prof_copy_rows.ncu-rep
