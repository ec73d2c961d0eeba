#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -u -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
bash scripts/pf_ab.sh > gpurun_out/pf_ab.txt 2>&1; cat gpurun_out/pf_ab.txt
