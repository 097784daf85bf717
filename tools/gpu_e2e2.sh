timeout 600 python -m pytest tests -q -m gpu -x -k "host or c1 or concurrent or Host" > gpurun_out/pytest_host.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_host.log
timeout 300 python tools/e2e_probe3.py
