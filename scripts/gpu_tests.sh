#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu_full.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_full.log
tail -n 15 gpurun_out/pytest_gpu_full.log
