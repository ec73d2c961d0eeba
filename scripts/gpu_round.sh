# One GPU session: GPU tests (x2), the bench line, the ncu launch list.
mkdir -p gpurun_out
for i in 1 2; do
  python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_$i.log 2>&1
  echo "rc=$?" >> gpurun_out/pytest_gpu_$i.log
done
python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "$1" = "ncu" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy_rows -s 81 -c 1 \
  -o gpurun_out/prof_copy_rows python profiles/drivers/migrate.py --reps 3 > gpurun_out/ncu_full.log 2>&1
fi
for f in gpurun_out/pytest_gpu_*.log; do tail -n 2 $f; done
