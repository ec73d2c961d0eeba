"""Profiling driver: one-layer and 80-layer DirectSend device time of the kernel movers (bench.measure_send_modes)."""
import sys, json
sys.path.insert(0, '.')
import torch, bench
bench.SEND_ARMS = [a for a in bench.SEND_ARMS if a[0] in ('kernel_full', 'kernel_32ctas')]
print(json.dumps(bench.measure_send_modes(torch)))
