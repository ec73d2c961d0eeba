#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 python -u -m pytest tests/test_layer_ready_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 900 python -u -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5
