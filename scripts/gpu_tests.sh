mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu_full.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_full.log
