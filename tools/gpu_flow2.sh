mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "sketch or c4 or Sketch or newton or Newton or multi_block" > gpurun_out/pytest_flow2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_flow2.log
for f in 2 1 0; do SPN_FLOW=$f timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e --no-check 2>&1 >/dev/null | tail -1 | sed "s/^/flow=$f /"; done
for g in 2 3 6 8; do SPN_FLOW_G=$g timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e --no-check 2>&1 >/dev/null | tail -1 | sed "s/^/flow=2 G=$g /"; done
