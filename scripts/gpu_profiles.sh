# ncu evidence for the current kernels: launch list of the default bench
# command, ncu --set full of the DirectSend copy and of decode attention.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy_rows -s 81 -c 1 \
  -o gpurun_out/prof_copy_rows python profiles/drivers/migrate.py --reps 3 > gpurun_out/ncu_full.log 2>&1
CASES=32x8192 REPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 3 -c 1 \
  -o gpurun_out/prof_decode python profiles/drivers/decode.py > gpurun_out/ncu_decode.log 2>&1
ls -la gpurun_out/*.ncu-rep
