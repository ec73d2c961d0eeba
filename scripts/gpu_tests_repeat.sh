mkdir -p gpurun_out
for i in 1 2 3 4; do
  python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_rep_$i.log 2>&1
  echo "rc=$?" >> gpurun_out/pytest_rep_$i.log
done
