#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_wire_gpu.py -x -q -p no:cacheprovider > gpurun_out/wire_tests.log 2>&1
timeout 300 python -u profiles/drivers/frames.py > gpurun_out/frames_driver.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_crc32 -s 50 -c 1 \
  -o gpurun_out/prof_crc32 -f python profiles/drivers/frames.py > gpurun_out/ncu_crc.log 2>&1
tail -n 5 gpurun_out/wire_tests.log; cat gpurun_out/frames_driver.log; tail -n 3 gpurun_out/ncu_crc.log
