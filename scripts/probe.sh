#!/bin/bash
cd "$(dirname "$0")/.."
for rep in 1 2 3; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(' value', d['value'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'], d.get('e2e_phases_us'))"
done
timeout 900 python -u -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
