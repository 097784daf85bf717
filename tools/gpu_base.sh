#!/bin/bash
# Baseline pass: -m gpu suite, smoke, default bench line.  usage: tools/gpu_base.sh tag
tag=${1:-x}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/smoke_$tag.log
timeout 1200 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"; tail -n 1 gpurun_out/bench_$tag.json | cut -c1-400
