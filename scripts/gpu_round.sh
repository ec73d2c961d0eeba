#!/bin/bash
# One GPU session: full GPU tests, the bench line, ncu launch list, ncu of
# the prefill kernel (tail case) and of k_first_nonfull.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
CASES=8192:6554 REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_prefill_attn -s 3 -c 1 \
  -o gpurun_out/prof_prefill -f python profiles/drivers/prefill.py > gpurun_out/ncu_prefill.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e'], d['roofline']['frac']); print(d.get('e2e_phases_us')); s=d['secondary']; print(s['transfer_sweep']['16'], s['configs']['70b_balanced_r0.2'], s['handoff'])"
