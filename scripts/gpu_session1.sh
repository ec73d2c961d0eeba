mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 300 python -u -m pytest tests/test_prefill_attention_gpu.py -x -q -p no:cacheprovider > gpurun_out/prefill_tests.log 2>&1
timeout 200 python -u profiles/drivers/prefill.py > gpurun_out/prefill_driver.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/prefill_tests.log; cat gpurun_out/prefill_driver.log | tail; tail -3 gpurun_out/pytest_gpu.log
