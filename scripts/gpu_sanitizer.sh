#!/bin/bash
# compute-sanitizer over the GPU tests (race detection / memory checking on the
# kernels): memcheck on the copy, send, relay, wire, attention and async tests; racecheck on the
# shared-memory kernels (decode page chunks, prefill, fan-out); synccheck on attention + parity.
cd "$(dirname "$0")/.."
O=gpurun_out/san
mkdir -p $O
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest \
  tests/test_gpu_parity.py tests/test_append_layers_gpu.py tests/test_boundary_safety_gpu.py \
  -q -p no:cacheprovider > $O/memcheck1.log 2>&1
timeout 2000 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest \
  tests/test_decode_attention_gpu.py tests/test_prefill_attention_gpu.py tests/test_relay_gpu.py \
  tests/test_append_send_gpu.py tests/test_layer_ready_gpu.py tests/test_async_gpu.py \
  tests/test_wire_gpu.py tests/test_send_modes_gpu.py tests/test_concurrency_gpu.py \
  -q -p no:cacheprovider > $O/memcheck2.log 2>&1
timeout 1000 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 --error-exitcode 9 \
  python -m pytest tests/test_decode_attention_gpu.py tests/test_prefill_attention_gpu.py \
  tests/test_append_send_gpu.py -q -p no:cacheprovider > $O/racecheck.log 2>&1
timeout 1000 compute-sanitizer --tool synccheck --print-limit 20 --error-exitcode 9 python -m pytest \
  tests/test_decode_attention_gpu.py tests/test_prefill_attention_gpu.py tests/test_gpu_parity.py \
  -q -p no:cacheprovider > $O/synccheck.log 2>&1
tail -n 3 $O/*.log
