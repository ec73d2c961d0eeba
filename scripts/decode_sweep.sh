mkdir -p gpurun_out
CASES=1x8192,4x8192,8x8192,32x8192,128x4096,8x32768,64x2048,256x1024 python profiles/drivers/decode.py > gpurun_out/decode_default.txt 2>&1
python -m pytest tests/test_decode_attention_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_decode.log 2>&1
cat gpurun_out/decode_default.txt; tail -n 3 gpurun_out/pytest_decode.log
