#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -u -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['secondary']
print(' value', d['value'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])
print(' sweep', {k: v['device_us'] for k, v in s['transfer_sweep'].items()})
print(' handoff', s['handoff']['exposed_tail_us'], s['handoff']['slowdown_pct'], 'tail append', s['configs']['70b_balanced_r0.2']['tail_append_us'])"
done
