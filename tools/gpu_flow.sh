mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "sketch or c4 or Sketch or newton or Newton or multi_block or family" > gpurun_out/pytest_flow.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_flow.log
for f in 1 0; do for g in 2; do SPN_FLOW=$f SPN_FLOW_G=$g timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e --no-check 2>&1 >/dev/null | tail -1 | sed "s/^/flow=$f G=$g /"; done; done
for g in 1 3 4 8; do SPN_FLOW_G=$g timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e --no-check 2>&1 >/dev/null | tail -1 | sed "s/^/flow=1 G=$g /"; done
timeout 300 ncu --metrics gpu__time_duration.sum --csv --log-file gpurun_out/dense_launches2.csv python tools/dense_probe.py > /dev/null 2>&1
grep -o '"[^"]*gemm[^"]*"\|"[^"]*sm100[^"]*"' gpurun_out/dense_launches2.csv | sort | uniq -c | head
