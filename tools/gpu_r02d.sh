mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_r02d.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r02d.log
for v in default twobar; do
  if [ $v = twobar ]; then export SPN_LIB=$PWD/paper_1610_06209_b200/_lib/variants/twobar/libspinners_b200.so; fi
  timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --no-e2e --no-check 2>&1 >/dev/null | tail -1 | sed "s/^/$v /"
done
