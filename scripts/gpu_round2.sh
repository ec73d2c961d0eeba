#!/bin/bash
# Round-2 evidence: full bench line, reference arm, launch list of the default
# bench command, ncu --set full of the DirectSend copy, of a per-layer append
# and of decode attention (B=8 ctx 8K and B=1 ctx 32K).
cd "$(dirname "$0")/.."
O=gpurun_out/r02
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 3 > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy_rows -s 81 -c 1 \
  -o $O/prof_copy_rows python profiles/drivers/migrate.py --reps 3 > $O/ncu_copy.log 2>&1
CASES=8x8192 REPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 3 -c 1 \
  -o $O/prof_decode_b8 python profiles/drivers/decode.py > $O/ncu_decode.log 2>&1
CASES=1x32768 REPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 3 -c 1 \
  -o $O/prof_decode_b1 python profiles/drivers/decode.py >> $O/ncu_decode.log 2>&1
ls -la $O
