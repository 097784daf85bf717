timeout 900 python -m pytest tests -q -m gpu -x -k "c3 or hash or Hash or config3 or peer or collision" > gpurun_out/pytest_c3.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_c3.log
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --no-e2e --no-check 2>&1 >/dev/null | tail -1
