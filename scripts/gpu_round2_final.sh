#!/bin/bash
# Round-2 closing evidence: the reference arm, the launch list of the default bench command,
# ncu --set full of the DirectSend copy (the headline kernel) and of the prefill kernel.
cd "$(dirname "$0")/.."
O=gpurun_out/r02f
mkdir -p $O
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy_rows -s 81 -c 1 \
  -o $O/prof_copy_rows python profiles/drivers/migrate.py --reps 3 > $O/ncu_copy.log 2>&1
CASES=8192:0 REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_prefill -s 2 -c 1 \
  -o $O/prof_prefill python profiles/drivers/prefill.py > $O/ncu_prefill.log 2>&1
ls -la $O
