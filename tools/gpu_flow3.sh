timeout 600 python -m pytest tests -q -m gpu -x -k "sketch or c4 or Sketch or newton or Newton or multi_block" > gpurun_out/pytest_flow3.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_flow3.log
for g in 2 3 4; do SPN_FLOW_G=$g timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e --no-check 2>&1 >/dev/null | tail -1 | sed "s/^/G=$g /"; done
