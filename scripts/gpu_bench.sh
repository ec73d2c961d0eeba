#!/bin/bash
# Bench line (all secondaries), launch list of the default bench command.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print({k: d[k] for k in ('value','e2e','roofline')}); print(json.dumps(d['secondary'].get('prefill_attention'))); print(json.dumps(d['secondary'].get('frames')))"
cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench.err
