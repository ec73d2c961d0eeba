#!/bin/bash
# GPU session: wire-format parity tests, CRC/frame timings, ncu of k_crc32,
# ncu of the prefill attention kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_wire_gpu.py -x -q -p no:cacheprovider > gpurun_out/wire_tests.log 2>&1
timeout 300 python -u profiles/drivers/frames.py > gpurun_out/frames_driver.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/frames_launches.csv \
  python profiles/drivers/frames.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_crc32 -s 50 -c 1 \
  -o gpurun_out/prof_crc32 -f python profiles/drivers/frames.py > gpurun_out/ncu_crc.log 2>&1
CASES=8192:6554 REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_prefill_attn -s 3 -c 1 \
  -o gpurun_out/prof_prefill -f python profiles/drivers/prefill.py > gpurun_out/ncu_prefill.log 2>&1
tail -5 gpurun_out/wire_tests.log; cat gpurun_out/frames_driver.log; tail -3 gpurun_out/ncu_crc.log gpurun_out/ncu_prefill.log
